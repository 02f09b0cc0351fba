// Micro-benchmark: TMA 2-D tile load throughput per SM (ring of S stages,
// one producer thread, one consumer thread releasing slots immediately).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_bench tma_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../paper_1802_07170_b200/csrc/ptx.cuh"

namespace cmt { unsigned long long g_launches = 0; }
using namespace cmt;

__global__ void __launch_bounds__(64, 1) tma_kernel(const __grid_constant__ CUtensorMap tm, int rows_box, int nloads,
                                                   int stages, int rows_total, long long* cycles, int suspend, int same) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int bytes = rows_box * 128;
  uint64_t* full = (uint64_t*)(smem + stages * bytes);
  uint64_t* empty = full + 16;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    int stage = 0; uint32_t phase = 0;
    for (int i = 0; i < nloads; ++i) {
      ptx::mbar_wait(&empty[stage], phase ^ 1);
      int row = same ? ((i / 16) * rows_box) % (rows_total - rows_box) : ((blockIdx.x * 7 + i) * rows_box) % (rows_total - rows_box);
      ptx::tma_load_2d(&tm, &full[stage], smem + stage * bytes, (i % 16) * 64, row);
      ptx::mbar_expect_tx(&full[stage], bytes);
      if (++stage == stages) { stage = 0; phase ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int stage = 0; uint32_t phase = 0;
    for (int i = 0; i < nloads; ++i) {
      if (suspend) ptx::mbar_wait(&full[stage], phase);
      else {
        uint32_t a = ptx::smem_u32(&full[stage]);
        uint32_t ok = 0;
        while (!ok) {
          asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(ok) : "r"(a), "r"(phase) : "memory");
        }
      }
      ptx::mbar_arrive(&empty[stage]);
      if (++stage == stages) { stage = 0; phase ^= 1; }
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  cudaDriverEntryPointQueryResult q;
  void* fnp = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  const int H = 1024;  // 16 k-blocks of 64 cols
  for (int same : {0, 1})
  for (int rows_total : {8192}) {  // 16 MB (L2-resident) and 2 GB (HBM)
    void* buf;
    cudaMalloc(&buf, (size_t)rows_total * H * 2);
    cudaMemset(buf, 0, (size_t)rows_total * H * 2);
    long long* cyc;
    cudaMalloc(&cyc, 1024 * 8);
    for (int rows_box : {64, 128, 256}) {
      CUtensorMap tm;
      cuuint64_t gdim[2] = {(cuuint64_t)H, (cuuint64_t)rows_total};
      cuuint64_t gstr[1] = {(cuuint64_t)H * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)rows_box};
      cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int stages : {6}) {
        for (int grid : {1, 64, 128}) {
          for (int suspend : {1}) {
            int bytes = rows_box * 128;
            size_t smem = 2048 + (size_t)stages * bytes;
            if (smem > 227 * 1024) continue;
            cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int nloads = 256;
            tma_kernel<<<grid, 64, smem>>>(tm, rows_box, nloads, stages, rows_total, cyc, suspend, same);
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            tma_kernel<<<grid, 64, smem>>>(tm, rows_box, nloads, stages, rows_total, cyc, suspend, same);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            std::vector<long long> c(grid);
            cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
            double avg = 0; for (auto x : c) avg += x; avg /= grid;
            double bytes_sm = (double)nloads * bytes;
            printf("same=%d %s box_rows=%3d stages=%d grid=%3d suspend=%d: %.1f cyc/load  %.1f B/clk/SM  total %.0f GB/s\n",
                   same, rows_total == 8192 ? "L2 " : "HBM", rows_box, stages, grid, suspend, avg / nloads,
                   bytes_sm / avg, bytes_sm * grid / (ms * 1e-3) / 1e9);
          }
        }
      }
    }
    cudaFree(buf);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(e));
}
