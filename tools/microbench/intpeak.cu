// Integer-pipe peak microbenchmark for the N-Queens roofline denominator.
//
// Measures the sustained thread-level int32 instruction rate of the ops the
// DFS loop is made of (LOP3 / SHF / IADD3 on the ALU pipe, IMAD on the FMA
// pipe, POPC) with many independent dependency chains per thread, all SMs
// busy, and reports the SM clock seen during the run (clock64 vs globaltimer).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o intpeak intpeak.cu
//   ./intpeak            -> one JSON line per op class
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CH = 8;        // independent chains per thread
constexpr int UNR = 8;       // chain steps per loop trip (amortises the loop branch)
constexpr int ITERS = 512;   // loop trips; each trip = CH * UNR ops

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

template <int OP>
__global__ void __launch_bounds__(512) k_ops(uint32_t* out, uint32_t seed, uint64_t* clk) {
  uint32_t x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = seed ^ (threadIdx.x * 2654435761u + i);
  uint32_t yy[UNR], zz[UNR];  // distinct operands per step: no LOP3/IMAD chain folding
#pragma unroll
  for (int u = 0; u < UNR; ++u) { yy[u] = seed * (7u + 2u * u) + 3u; zz[u] = seed * (13u + 4u * u) + 5u; }
  uint64_t c0 = 0, t0 = 0;
  if (threadIdx.x == 0 && blockIdx.x == 0) { c0 = clock64(); t0 = gtimer(); }
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const uint32_t y = yy[u], z = zz[u];
      if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
      if (OP == 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(y), "r"(z));
      if (OP == 2) {  // 1:1 ALU:FMA mix
        if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(y), "r"(z));
        else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
      }
      if (OP == 3) asm volatile("popc.b32 %0, %0;" : "+r"(x[i]));
      if (OP == 4) asm volatile("shf.r.clamp.b32 %0, %0, %1, 1;" : "+r"(x[i]) : "r"(y));
      if (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(y));
      if (OP == 6) {  // 2 ALU : 1 FMA
        if (i % 3 == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(y), "r"(z));
        else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
      }
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = clock64() - c0; clk[1] = gtimer() - t0; }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) acc ^= x[i];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int OP>
int run(const char* name, int sms) {
  const int threads = 512, blocks = sms * 4;  // 2048 threads / SM
  uint32_t* out; uint64_t* clk;
  CK(cudaMalloc(&out, sizeof(uint32_t) * threads * blocks));
  CK(cudaMalloc(&clk, 16));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) k_ops<OP><<<blocks, threads>>>(out, 1u + w, clk);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  uint64_t hc[2] = {0, 0};
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_ops<OP><<<blocks, threads>>>(out, 7u + r, clk);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) { best = ms; CK(cudaMemcpy(hc, clk, 16, cudaMemcpyDeviceToHost)); }
  }
  const double ops = double(threads) * blocks * ITERS * CH * UNR;
  const double rate = ops / (best * 1e-3);
  const double mhz = hc[1] ? double(hc[0]) / double(hc[1]) * 1e3 : 0.0;
  const double per_sm_clk = rate / (sms * mhz * 1e6);
  printf("{\"op\": \"%s\", \"thread_ops_per_s\": %.4e, \"ms\": %.3f, \"sm_mhz\": %.0f, "
         "\"thread_ops_per_sm_clk\": %.1f}\n", name, rate, best, mhz, per_sm_clk);
  cudaFree(out); cudaFree(clk);
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"device\": \"%s\", \"sms\": %d, \"smem_per_sm\": %zu, \"smem_optin_per_block\": %zu, "
         "\"regs_per_sm\": %d}\n", p.name, p.multiProcessorCount, p.sharedMemPerMultiprocessor,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  const int sms = p.multiProcessorCount;
  run<0>("lop3", sms);
  run<1>("imad", sms);
  run<2>("lop3+imad 1:1", sms);
  run<3>("popc", sms);
  run<4>("shf", sms);
  run<5>("add.u32", sms);
  run<6>("lop3+imad 2:1", sms);
  return 0;
}
