// Probe: tcgen05.mma kind::f16 with the A operand in TMEM (M=128, N=64, K=64).
// A[m][k] is written to TMEM with tcgen05.st (lane m, bf16 pairs (2c, 2c+1) in
// column c); B[n][k] sits K-major, 128B-swizzled in smem.  D is compared with
// a host fp32 reference.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_1802_07170_b200/csrc/ptx.cuh"

using namespace cmt;

__device__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}

__global__ void probe(const bf16* A, const bf16* B, float* D, int N) {
  __shared__ __align__(1024) uint8_t sB[64 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B[n][k] -> smem row n (128 B), 16-byte chunk j at j ^ (n & 7)
  for (int i = threadIdx.x; i < N * 8; i += blockDim.x) {
    int n = i >> 3, j = i & 7;
    *(uint4*)(sB + n * 128 + ((j ^ (n & 7)) << 4)) = *(const uint4*)(B + n * 64 + j * 8);
  }
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 256);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t ta = tmem, td = tmem + 128;
  {  // row m = 32 warp + lane: 32 columns of bf16 pairs
    const int m = warp * 32 + lane;
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) {
      __nv_bfloat162 p;
      p.x = A[m * 64 + 2 * c];
      p.y = A[m * 64 + 2 * c + 1];
      r[c] = *(uint32_t*)&p;
    }
    tmem_st32(ta + ((uint32_t)(warp * 32) << 16), r);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_bf16(128, N, 0, 0);
    for (int kk = 0; kk < 4; ++kk) {
      uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(sB) + kk * 32, 16, 1024);
      umma_ts(td, ta + kk * 8, bd, idesc, kk ? 1u : 0u);
    }
    ptx::umma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  {
    const int m = warp * 32 + lane;
    float v[32];
    for (int c0 = 0; c0 < N; c0 += 32) {
      ptx::tmem_ld32(td + ((uint32_t)(warp * 32) << 16) + c0, v);
      for (int c = 0; c < 32 && c0 + c < N; ++c) D[m * N + c0 + c] = v[c];
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 256);
}


// MMA issue/execute rate: R rounds of 64 MMAs (M=128, N, K=16 each) with A
// from TMEM (mode 0) or from smem (mode 1, MN-major 128B atoms), B from smem.
template <int N>
__global__ void rate(int mode, int nacc, int R, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)dsm + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;               // 16 KB
  uint8_t* sB = sm + 16384;       // N x 128 B (N <= 256)
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_barrier_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t id_t = ptx::idesc_bf16(128, N, 0, 0), id_s = ptx::idesc_bf16(128, N, 1, 0);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      for (int i = 0; i < 64; ++i) {
        uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(sB) + (i & 3) * 32, 16, 1024);
        const uint32_t d = tmem + (uint32_t)((i % nacc) * N);  // nacc independent accumulators
        if (mode == 0) umma_ts(d, tmem + 256 + (i & 31) * 8, bd, id_t, 1u);
        else ptx::umma_bf16(d, ptx::smem_desc_sw128(ptx::smem_u32(sA) + (i & 3) * 2048, 8192, 1024), bd, id_s, 1u);
      }
      ptx::umma_commit(&bar);
      ptx::mbar_wait(&bar, r & 1);
    }
    cyc[0] = clock64() - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  const int M = 128, N = 64, K = 64;
  std::vector<bf16> hA(M * K), hB(N * K);
  std::vector<float> fA(M * K), fB(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) { hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < N * K; ++i) { hB[i] = __float2bfloat16((rand() % 17 - 8) / 8.f); fB[i] = __bfloat162float(hB[i]); }
  bf16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  probe<<<1, 128>>>(dA, dB, dD, N);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> hD(M * N);
  cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += fA[m * K + k] * fB[n * K + k];
      double err = fabs(r - hD[m * N + n]);
      if (err > 1e-3) { if (bad < 5) printf("m=%d n=%d ref=%f got=%f\n", m, n, r, hD[m * N + n]); ++bad; }
      maxerr = fmax(maxerr, err);
    }
  printf("TMEM-A probe: %s (max err %g, %d bad of %d)\n", bad ? "MISMATCH" : "OK", maxerr, bad, M * N);
  long long* dc;
  cudaMalloc(&dc, 8);
  cudaFuncSetAttribute(rate<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
  cudaFuncSetAttribute(rate<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
  cudaFuncSetAttribute(rate<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
  cudaFuncSetAttribute(rate<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int R = 4000;
  auto run = [&](int n, int mode, int nacc) {
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (n == 32) rate<32><<<1, 128, 60000>>>(mode, nacc, R, dc);
      if (n == 64) rate<64><<<1, 128, 60000>>>(mode, nacc, R, dc);
      if (n == 128) rate<128><<<1, 128, 60000>>>(mode, nacc, R, dc);
      if (n == 256) rate<256><<<1, 128, 60000>>>(mode, nacc, R, dc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    long long c = 0;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    double ns = ms * 1e6 / (R * 64.0);
    printf("A %s N=%3d acc=%d: %.1f ns/MMA (%.1f clk64/MMA)  %.2f TFLOP/s per SM\n", mode ? "smem" : "TMEM", n, nacc, ns,
           c / (R * 64.0), 2.0 * 128 * n * 16 / ns / 1e3);
  };
  for (int n : {32, 64, 128, 256}) run(n, 1, 1);
  for (int n : {32, 64, 128}) run(n, 0, 1);
  run(64, 1, 4);
  run(64, 0, 4);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return bad ? 2 : 0;
}
