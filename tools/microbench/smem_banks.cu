// smem_banks.cu — how sm_100 counts shared-memory wavefronts and bank conflicts for
// predicated 16-byte accesses to the DFS stack layout (frame L of thread t at
// stk[L*BLOCK + t]). Each pattern is one kernel launch; profile with
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,\
//     l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,\
//     l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,\
//     l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,\
//     smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum ./smem_banks
// and divide by the instruction counts.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int BLOCK = 128, LEVELS = 16, ITERS = 1024;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// mode: bit0 = random level per lane (else level 0); bits1-2: active set
//   0 = all lanes, 1 = ~37% random, 2 = lanes {0, 8}, 3 = lanes {0, 1};
//   bit3: padded rows (level stride BLOCK+1 frames: lane t's bank group rotates with L)
template <int MODE, bool LOAD>
__global__ void __launch_bounds__(BLOCK) pattern(uint32_t* out, uint32_t seed) {
  __shared__ uint4 stk[LEVELS * (BLOCK + 1)];
  const uint32_t t = threadIdx.x, lane = t & 31u;
  for (int i = t; i < LEVELS * (BLOCK + 1); i += BLOCK) stk[i] = make_uint4(i, i, i, i);
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(stk)) + t * 16u;
  uint32_t acc = 0;
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
    const uint32_t h = hash(seed ^ (it * 131u) ^ (t * 7919u));
    const uint32_t level = (MODE & 1) ? (h % LEVELS) : 0u;
    bool active;
    switch ((MODE >> 1) & 3) {
      case 0: active = true; break;
      case 1: active = (h >> 8) % 100u < 37u; break;
      case 2: active = lane == 0u || lane == 8u; break;
      default: active = lane == 0u || lane == 1u; break;
    }
    const uint32_t addr = base + level * ((MODE & 8) ? (BLOCK + 1) : BLOCK) * 16u;
    if (LOAD) {
      uint32_t x = 0, y = 0, z = 0, w = 0;
      asm volatile(
          "{ .reg .pred p; setp.ne.u32 p, %5, 0;\n\t"
          "@p ld.shared.v4.u32 {%0, %1, %2, %3}, [%4]; }"
          : "+r"(x), "+r"(y), "+r"(z), "+r"(w)
          : "r"(addr), "r"(active ? 1u : 0u)
          : "memory");
      acc += x ^ y ^ z ^ w;
    } else {
      asm volatile(
          "{ .reg .pred p; setp.ne.u32 p, %1, 0;\n\t"
          "@p st.shared.v4.u32 [%0], {%2, %2, %2, %2}; }" ::"r"(addr),
          "r"(active ? 1u : 0u), "r"(h)
          : "memory");
    }
  }
  if (acc == 0x12345u) out[t] = acc;
}

template <int MODE>
void run(uint32_t* out) {
  pattern<MODE, true><<<1, BLOCK>>>(out, 1);
  pattern<MODE, false><<<1, BLOCK>>>(out, 1);
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 4096);
  run<0>(out);  // all lanes, same level
  run<1>(out);  // all lanes, random levels
  run<2>(out);  // 37% lanes, same level
  run<3>(out);  // 37% lanes, random levels
  run<4>(out);  // lanes {0,8}, same level
  run<5>(out);  // lanes {0,8}, random levels
  run<6>(out);  // lanes {0,1}, same level
  run<7>(out);  // lanes {0,1}, random levels
  run<11>(out);  // padded: 37% lanes, random levels
  run<13>(out);  // padded: lanes {0,8}, random levels
  run<9>(out);   // padded: all lanes, random levels
  cudaDeviceSynchronize();
  std::printf("patterns done: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
