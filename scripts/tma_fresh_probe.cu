// Does a TMA load of data another SM has JUST written (the recurrent scans'
// h_t / dU_t exchange) take longer than a load of the same bytes read again?
// CTA 0 (producer) writes a 128 KB block (generic st.global, or a bulk TMA
// store from smem), then releases a flag; CTA 1 (consumer) acquires it and
// TMA-loads the block as 4 x 32 KB 2-D boxes, timing issue -> complete, then
// loads it a second time.  Repeats 64 rounds; prints medians (ns).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1802_07170_b200/csrc -o scripts/tma_fresh_probe scripts/tma_fresh_probe.cu -lcuda
#include <cuda.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "ptx.cuh"

using namespace cmt;
constexpr int ROWS = 256, COLS = 256;  // bf16 [256][256] = 128 KB, 4 boxes of [64 rows][256]... as [rows][64] tiles
constexpr int ROUNDS = 64;

__device__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void probe(const __grid_constant__ CUtensorMap tm, bf16* X, unsigned* flag, unsigned long long* out,
                      int mode, int nc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int r = 0; r < ROUNDS; ++r) {
    if (blockIdx.x == 0) {  // producer
      if (r > 0) {
        if (tid == 0)
          while (ptx::ld_acquire(flag + 1) < (unsigned)(r * nc)) {
          }
        __syncthreads();
      }
      if (mode != 2) {  // mode 2: never rewritten (stale data every round)
        for (int i = tid; i < ROWS * COLS / 8; i += blockDim.x) {
          uint4 v = make_uint4(r, i, r ^ i, 7);
          ((uint4*)X)[i] = v;
        }
      }
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(flag, 1u);
      }
    } else {  // consumer
      if (tid == 0) {
        while (ptx::ld_acquire(flag) < (unsigned)(r + 1)) {
        }
        ptx::fence_proxy_async_global();
        for (int pass = 0; pass < 2; ++pass) {
          const unsigned long long t0 = gt();
          ptx::mbar_expect_tx(&bar, ROWS * COLS * 2);
          for (int q = 0; q < COLS / 64; ++q)
            for (int h = 0; h < ROWS / 128; ++h)
              ptx::tma_load_2d(&tm, &bar, sm + (q * (ROWS / 128) + h) * 16384, q * 64, h * 128);
          ptx::mbar_wait(&bar, phase);
          phase ^= 1;
          if (blockIdx.x == 1) out[(r * 2 + pass)] = gt() - t0;
        }
        atomicAdd(flag + 1, 1u);
      }
      __syncthreads();
    }
  }
}

int main(int argc, char** argv) {
  const int nc = argc > 1 ? atoi(argv[1]) : 1;  // consumer CTAs reading the same block
  bf16* X;
  unsigned* flag;
  unsigned long long* out;
  cudaMalloc(&X, ROWS * COLS * 2);
  cudaMalloc(&flag, 8);
  cudaMalloc(&out, ROUNDS * 2 * 8);
  cudaMemset(X, 0, ROWS * COLS * 2);
  CUtensorMap tm;
  cuuint64_t gdim[2] = {COLS, ROWS};
  cuuint64_t gstr[1] = {COLS * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 140 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"fresh (rewritten every round)", "fresh, second read", "stale (never rewritten)"};
  for (int mode : {0, 2}) {
    cudaMemset(flag, 0, 8);
    probe<<<1 + nc, 256, smem>>>(tm, X, flag, out, mode, nc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<unsigned long long> h(ROUNDS * 2);
    cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
    std::vector<unsigned long long> a, b;
    for (int r = 4; r < ROUNDS; ++r) { a.push_back(h[2 * r]); b.push_back(h[2 * r + 1]); }
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    printf("consumers %d, mode %d: 128 KB TMA load, first read %llu ns (%s), second read %llu ns (%s)\n", nc, mode, a[a.size() / 2],
           mode == 0 ? names[0] : names[2], b[b.size() / 2], mode == 0 ? names[1] : names[2]);
  }
  return 0;
}
