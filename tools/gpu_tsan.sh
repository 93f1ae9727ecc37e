# Host-side race detection of the scheduler / checkpoint threads (ThreadSanitizer on the
# C++ drop-in test; the CUDA driver's own internals are suppressed).
mkdir -p gpurun_out
cat > /tmp/tsan.supp <<'SUPP'
called_from_lib:libcuda.so
called_from_lib:libcudart.so
race:libcuda.so
SUPP
g++ -O1 -g -std=c++20 -fsanitize=thread -Iinclude -o /tmp/test_dropin_tsan tests/cpp/test_dropin.cpp \
  -Lpaper_2511_12009_b200 -l:libnqb200.so -Wl,-rpath,$PWD/paper_2511_12009_b200 -pthread
TSAN_OPTIONS="suppressions=/tmp/tsan.supp halt_on_error=0 report_signal_unsafe=0" timeout 900 /tmp/test_dropin_tsan gpu > gpurun_out/tsan.log 2>&1
echo "rc=$?" >> gpurun_out/tsan.log
grep -c "WARNING: ThreadSanitizer" gpurun_out/tsan.log; tail -5 gpurun_out/tsan.log
