// Which SMs sit on which die, and what a cross-die flag round trip costs.
// One CTA per SM (large dynamic smem).  Turn by turn (a global ticket), each
// CTA times 256 dependent atomics on each of several global addresses; an
// address's L2 home slice sits on one die, so SMs on that die see the short
// latency.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/die_probe scripts/die_probe.cu
#include <cstdio>
#include <vector>

constexpr int NADDR = 8;
__global__ void probe(unsigned* flags, unsigned* ticket, long long* out, int* smid_out) {
  extern __shared__ char pad[];
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  pad[0] = 0;
  if (threadIdx.x != 0) return;
  // take a turn
  const unsigned me = atomicAdd(ticket, 1u);
  while (atomicAdd(ticket + 1, 0u) != me) {
  }
  smid_out[me] = (int)sm;
  for (int a = 0; a < NADDR; ++a) {
    unsigned* p = flags + a * 4096;  // 16 KB apart: different L2 slices
    unsigned v = 0;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) v = atomicAdd(p + (v >> 30), 1u);  // dependent: v stays small
    long long t1 = clock64();
    out[me * NADDR + a] = (t1 - t0) / 256 + (v >> 30);
  }
  __threadfence();
  atomicAdd(ticket + 1, 1u);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned *flags, *ticket;
  long long* out;
  int* smid;
  cudaMalloc(&flags, NADDR * 4096 * 4);
  cudaMalloc(&ticket, 8);
  cudaMalloc(&out, nsm * NADDR * 8);
  cudaMalloc(&smid, nsm * 4);
  cudaMemset(flags, 0, NADDR * 4096 * 4);
  cudaMemset(ticket, 0, 8);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  void* args[] = {&flags, &ticket, &out, &smid};
  cudaLaunchCooperativeKernel((void*)probe, nsm, 32, args, smem, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<long long> h(nsm * NADDR);
  std::vector<int> s(nsm);
  cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(s.data(), smid, s.size() * 4, cudaMemcpyDeviceToHost);
  std::vector<std::vector<long long>> by(nsm, std::vector<long long>(NADDR));
  for (int i = 0; i < nsm; ++i)
    for (int a = 0; a < NADDR; ++a) by[s[i]][a] = h[i * NADDR + a];
  printf("smid: atomic round-trip cycles for %d addresses\n", NADDR);
  for (int m = 0; m < nsm; ++m) {
    printf("%3d:", m);
    for (int a = 0; a < NADDR; ++a) printf(" %5lld", by[m][a]);
    printf("\n");
  }
  return 0;
}
