// Issue-to-completion time of a chain of n tcgen05.mma (kind::f16, M=128, K=16 each)
// on one SM, A from shared memory (MN-major, as the scans' smem-resident W_h
// k-blocks) or from TMEM (the scans' TMEM-resident k-blocks), B K-major in
// shared memory, N = 64 / 128 / 256.  One thread issues, commits once and waits
// on the mbarrier.  Prints cycles for n = 1, 16, 64, 256 and the per-MMA slope,
// against the floor 128*N*16 MACs / 2831 MAC/clk/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1802_07170_b200/csrc -o scripts/mma_rate_probe scripts/mma_rate_probe.cu
#include <cstdio>
#include "ptx.cuh"

using namespace cmt;

__device__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}

// whole-warp issue: every lane runs the loop with uniform values, one elected lane issues
__device__ void umma_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ void umma_ss_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ void commit_w(uint64_t* bar) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
               ::"r"(ptx::smem_u32(bar)) : "memory");
}

__global__ void probe_w(long long* out, int N, int a_tmem) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sA = sm;
  uint8_t* sB = sm + 4 * 16384;
  for (int i = threadIdx.x; i < (4 * 16384 + 4 * N * 128) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t tA = tbase + 256;
  uint32_t phase = 0;
  if (threadIdx.x < 32) {  // the whole warp
    const uint32_t idesc_s = ptx::idesc_bf16(128, N, 1, 0);
    const uint32_t idesc_t = ptx::idesc_bf16(128, N, 0, 0);
    const uint32_t abase = ptx::smem_u32(sA), bbase = ptx::smem_u32(sB);
    const int counts[4] = {1, 16, 64, 256};
    for (int rep = 0; rep < 2; ++rep)
      for (int ci = 0; ci < 4; ++ci) {
        const int n = counts[ci];
        __syncwarp();
        const long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
          const int kb = (i >> 2) & 3, kk = i & 3;
          const uint64_t bd = ptx::smem_desc_sw128(bbase + kb * N * 128 + kk * 32, 16, 1024);
          if (a_tmem) {
            umma_ts_w(tmem, tA + (uint32_t)(((i >> 2) & 7) * 32 + kk * 8), bd, idesc_t, i > 0);
          } else {
            const uint64_t ad = ptx::smem_desc_sw128(abase + kb * 16384 + kk * 2048, 8192, 1024);
            umma_ss_w(tmem, ad, bd, idesc_s, i > 0);
          }
        }
        commit_w(&bar);
        ptx::mbar_wait(&bar, phase);
        phase ^= 1;
        const long long t1 = clock64();
        if (rep == 1 && threadIdx.x == 0) out[ci] = t1 - t0;
      }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tbase, 512);
}

// fully unrolled issue with precomputed descriptors (base + constant offsets)
template <int NM>
__device__ __forceinline__ void issue_unrolled(uint32_t tmem, uint32_t tA, uint64_t ad0, uint64_t bd0, uint32_t idesc,
                                               int a_tmem, int N) {
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    const int kb = (i >> 2) & 3, kk = i & 3;
    const uint64_t bd = bd0 + (uint64_t)((kb * N * 128 + kk * 32) >> 4);
    if (a_tmem) {
      umma_ts_w(tmem, tA + (uint32_t)(((i >> 2) & 7) * 32 + kk * 8), bd, idesc, i > 0);
    } else {
      const uint64_t ad = ad0 + (uint64_t)((kb * 16384 + kk * 2048) >> 4);
      umma_ss_w(tmem, ad, bd, idesc, i > 0);
    }
  }
}
__global__ void probe_u(long long* out, int N, int a_tmem) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* sA = sm;
  uint8_t* sB = sm + 4 * 16384;
  for (int i = threadIdx.x; i < (4 * 16384 + 4 * N * 128) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t tA = tbase + 256;
  uint32_t phase = 0;
  if (threadIdx.x < 32) {
    const uint32_t idesc = a_tmem ? ptx::idesc_bf16(128, N, 0, 0) : ptx::idesc_bf16(128, N, 1, 0);
    const uint64_t ad0 = ptx::smem_desc_sw128(ptx::smem_u32(sA), 8192, 1024);
    const uint64_t bd0 = ptx::smem_desc_sw128(ptx::smem_u32(sB), 16, 1024);
    for (int rep = 0; rep < 2; ++rep)
      for (int ci = 0; ci < 3; ++ci) {
        __syncwarp();
        const long long t0 = clock64();
        if (ci == 0) issue_unrolled<16>(tmem, tA, ad0, bd0, idesc, a_tmem, N);
        else if (ci == 1) issue_unrolled<64>(tmem, tA, ad0, bd0, idesc, a_tmem, N);
        else issue_unrolled<128>(tmem, tA, ad0, bd0, idesc, a_tmem, N);
        commit_w(&bar);
        ptx::mbar_wait(&bar, phase);
        phase ^= 1;
        const long long t1 = clock64();
        if (rep == 1 && threadIdx.x == 0) out[ci] = t1 - t0;
      }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tbase, 512);
}

__global__ void probe(long long* out, int N, int a_tmem, int chains) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  // A: 16 k-blocks x [64 k][128 m] (16 KB each) = 256 KB is too much: reuse 4 k-blocks
  uint8_t* sA = sm;               // 4 x 16 KB
  uint8_t* sB = sm + 4 * 16384;   // 4 x [N rows][64 k] bf16 (N*128 B each)
  for (int i = threadIdx.x; i < (4 * 16384 + 4 * N * 128) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;       // D: columns [0, N)
  const uint32_t tA = tbase + 256;   // A in TMEM: columns [256, 512)
  uint32_t phase = 0;
  if (threadIdx.x == 0) {
    const uint32_t idesc_s = ptx::idesc_bf16(128, N, 1, 0);
    const uint32_t idesc_t = ptx::idesc_bf16(128, N, 0, 0);
    const uint32_t abase = ptx::smem_u32(sA), bbase = ptx::smem_u32(sB);
    const int counts[4] = {1, 16, 64, 256};
    for (int rep = 0; rep < 2; ++rep)
      for (int ci = 0; ci < 4; ++ci) {
        const int n = counts[ci];
        const long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
          const int kb = (i >> 2) & 3, kk = i & 3;
          const uint64_t bd = ptx::smem_desc_sw128(bbase + kb * N * 128 + kk * 32, 16, 1024);
          const uint32_t dcol = tmem + (uint32_t)((i % chains) * N);  // independent accumulators
          const uint32_t acc = i >= chains;
          if (a_tmem) {
            umma_ts(dcol, tA + (uint32_t)(((i >> 2) & 7) * 32 + kk * 8), bd, idesc_t, acc);
          } else {
            const uint64_t ad = ptx::smem_desc_sw128(abase + kb * 16384 + kk * 2048, 8192, 1024);
            ptx::umma_bf16(dcol, ad, bd, idesc_s, acc);
          }
        }
        ptx::umma_commit(&bar);
        ptx::mbar_wait(&bar, phase);
        phase ^= 1;
        const long long t1 = clock64();
        if (rep == 1) out[ci] = t1 - t0;
      }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x < 32) ptx::tmem_dealloc(tbase, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  const int smem = 4 * 16384 + 4 * 256 * 128 + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe_w, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe_u, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
    for (int N : {64, 128, 256}) {
      probe_u<<<1, 128, smem>>>(d, N, a_tmem);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[4];
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("unrolled A %-4s N=%3d: n=16 %5lld  n=64 %6lld  n=128 %6lld cyc; slope %.1f cyc/MMA\n",
             a_tmem ? "tmem" : "smem", N, h[0], h[1], h[2], (h[2] - h[1]) / 64.0);
    }
  for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
    for (int N : {64, 128, 256}) {
      probe_w<<<1, 128, smem>>>(d, N, a_tmem);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[4];
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("warp-issue A %-4s N=%3d: n=1 %5lld  n=16 %5lld  n=64 %6lld  n=256 %6lld cyc; slope %.1f cyc/MMA\n",
             a_tmem ? "tmem" : "smem", N, h[0], h[1], h[2], h[3], (h[3] - h[2]) / 192.0);
    }
  for (int chains : {1, 2})
  for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
    for (int N : {64, 128, 256}) {
      if (N * chains > 256) continue;
      probe<<<1, 128, smem>>>(d, N, a_tmem, chains);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[4];
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("chains %d A %-4s N=%3d: n=1 %5lld  n=16 %5lld  n=64 %6lld  n=256 %6lld cyc; slope %.1f cyc/MMA (floor %.1f)\n",
             chains, a_tmem ? "tmem" : "smem", N, h[0], h[1], h[2], h[3], (h[3] - h[2]) / 192.0, 128.0 * N * 16 / 2831.0);
    }
  return 0;
}
