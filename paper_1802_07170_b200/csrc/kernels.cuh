// Memory-bound and small fused kernels of the train step: embedding gather /
// deterministic scatter, PCG64-exact dropout, bidirectional sum, Luong
// attention forward/backward, fused log-softmax + label-smoothed CE + grad,
// column sums (bias grads), global-norm reduction and the clipped SGD update.
#pragma once
#include <cmath>
#include "common.cuh"

namespace cmt {

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
template <typename T>
CMT_D float ldf(const T* p, long long i) { return to_f<T>(p[i]); }

CMT_D float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
CMT_D float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
CMT_D double warp_sumd(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// Embedding (reference tensor.py:191-216, layers.py:79-113)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ table, int E, const int* __restrict__ ids, int N,
                                   T* __restrict__ out) {
  int n = blockIdx.x;
  if (n >= N) return;
  const T* src = table + (long long)ids[n] * E;
  T* dst = out + (long long)n * E;
  if (((E * sizeof(T)) & 15) == 0 && (((uintptr_t)table | (uintptr_t)out) & 15) == 0) {  // 16-byte rows
    const int nv = (int)(E * sizeof(T) / 16);
    for (int e = threadIdx.x; e < nv; e += blockDim.x) ((uint4*)dst)[e] = __ldg((const uint4*)src + e);
    return;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) dst[e] = src[e];
}

// gout[u][:] = sum over positions p of segment u (in position order) of dX[pos[p]][:]
// — the deterministic equivalent of np.add.at(table_grad, ids, dX.T).
__global__ void scatter_compact_kernel(const float* __restrict__ dX, int E, const int* __restrict__ seg_off,
                                       const int* __restrict__ seg_pos, int nseg, float* __restrict__ gout,
                                       const int* __restrict__ nseg_d = nullptr) {
  int u = blockIdx.x;
  if (nseg_d) nseg = *nseg_d;
  if (u >= nseg) return;
  const int b = seg_off[u], e_ = seg_off[u + 1];
  // up to 8 columns per thread and 4 positions per iteration in flight (long
  // segments such as BOS span every sentence); fixed summation order, so the
  // result is deterministic (4 interleaved partial sums, combined in order)
  for (int e0 = threadIdx.x; e0 < E; e0 += 8 * blockDim.x) {
    float acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[r][j] = 0.f;
    int p = b;
    for (; p + 4 <= e_; p += 4) {
      long long rowp[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) rowp[r] = (long long)seg_pos[p + r] * E;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int e = e0 + j * blockDim.x;
          if (e < E) acc[r][j] += dX[rowp[r] + e];
        }
    }
    for (; p < e_; ++p) {
      const long long rp = (long long)seg_pos[p] * E;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = e0 + j * blockDim.x;
        if (e < E) acc[0][j] += dX[rp + e];
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = e0 + j * blockDim.x;
      if (e < E) gout[(long long)u * E + e] = (acc[0][j] + acc[1][j]) + (acc[2][j] + acc[3][j]);
    }
  }
}

// E % 4 == 0 variant: one float4 column group per thread, the segment's
// positions staged 8 at a time, 8 rows in flight per thread.  Summation order
// is fixed (8 interleaved partials combined as a tree), so it is deterministic.
constexpr int SCAT_THREADS = 256;
__global__ void __launch_bounds__(SCAT_THREADS) scatter_compact_v4_kernel(const float* __restrict__ dX, int E,
                                                                          const int* __restrict__ seg_off,
                                                                          const int* __restrict__ seg_pos, int nseg,
                                                                          float* __restrict__ gout,
                                                                          const int* __restrict__ nseg_d = nullptr) {
  const int u = blockIdx.x;
  if (nseg_d) nseg = *nseg_d;  // the count from the step scalars (grid sized for the bucket's maximum)
  if (u >= nseg) return;
  const int b = seg_off[u], e_ = seg_off[u + 1];
  const int E4 = E >> 2;
  for (int c = threadIdx.x; c < E4; c += blockDim.x) {
    float4 acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p = b; p < e_; p += 8) {
      int pos[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) pos[r] = p + r < e_ ? __ldg(seg_pos + p + r) : -1;
      float4 v[8];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        v[r] = pos[r] >= 0 ? __ldg((const float4*)(dX + (long long)pos[r] * E) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        acc[r].x += v[r].x; acc[r].y += v[r].y; acc[r].z += v[r].z; acc[r].w += v[r].w;
      }
    }
#pragma unroll
    for (int w = 4; w; w >>= 1)
#pragma unroll
      for (int r = 0; r < w; ++r) {
        acc[r].x += acc[r + w].x; acc[r].y += acc[r + w].y; acc[r].z += acc[r + w].z; acc[r].w += acc[r + w].w;
      }
    ((float4*)(gout + (long long)u * E))[c] = acc[0];
  }
}

// ---------------------------------------------------------------------------
// Embedding segments on the device, equal to the host staging path's result:
// the positions of one table's ids sorted stably by id (LSD radix, 4-bit
// digits; positions stay ascending within an id = np.add.at order), the
// unique ids in ascending order, their segment offsets and their count.  One
// CTA of SEG_THREADS per table: positions in shared memory (two buffers),
// per-thread digit counts as 16-bit counters, chunks of consecutive elements
// per thread so the scatter is stable.
// ---------------------------------------------------------------------------
constexpr int SEG_THREADS = 1024;
constexpr int SEG_MAX_N = 24576;  // elements per table (offsets fit 16 bits)
struct SegJob {
  const int* ids0;  // positions [0, n0): ids0[p]
  const int* ids1;  // positions [n0, n0 + n1): ids1[p - n0]
  int n0, n1, pos_base;
  int* off;    // [nu + 1]
  int* pos;    // [n] global positions, grouped by id
  int* uq;     // [nu] ascending unique ids
  int* nrows;  // nu
};
inline size_t seg_smem(int n) { return (size_t)2 * n * 4 + (size_t)16 * SEG_THREADS * 2 + 48 * 4; }
// exclusive prefix sum over the CTA (SEG_THREADS threads); *total = the sum
CMT_D int seg_excl_scan(int v, int* sh, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    const int s0 = sh[lane];
    int t = s0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    sh[lane] = t - s0;
    if (lane == 31) sh[32] = t;
  }
  __syncthreads();
  const int r = sh[w] + x - v;
  *total = sh[32];
  __syncthreads();
  return r;
}
__global__ void __launch_bounds__(SEG_THREADS) segments_kernel(SegJob j0, SegJob j1, int bits) {
  const SegJob J = blockIdx.x ? j1 : j0;
  const int n = J.n0 + J.n1;
  extern __shared__ int segsm[];
  int* A = segsm;
  int* Bf = A + n;
  unsigned short* hist = (unsigned short*)(Bf + n);  // [16][SEG_THREADS]
  int* sh = (int*)(hist + 16 * SEG_THREADS);
  const int t = threadIdx.x;
  auto idof = [&](int p) { return p < J.n0 ? __ldg(J.ids0 + p) : __ldg(J.ids1 + (p - J.n0)); };
  const int c = (n + SEG_THREADS - 1) / SEG_THREADS;
  const int b0 = min(n, t * c), b1 = min(n, b0 + c);
  for (int i = t; i < n; i += SEG_THREADS) A[i] = i;
  __syncthreads();
  for (int shift = 0; shift < bits; shift += 4) {
#pragma unroll
    for (int d = 0; d < 16; ++d) hist[d * SEG_THREADS + t] = 0;
    for (int i = b0; i < b1; ++i) ++hist[((idof(A[i]) >> shift) & 15) * SEG_THREADS + t];
    __syncthreads();
    // exclusive offsets over the digit-major order (digit, thread): thread t owns entries [16 t, 16 t + 16)
    int loc[16], sum = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      loc[k] = sum;
      sum += hist[16 * t + k];
    }
    int tot;
    const int base = seg_excl_scan(sum, sh, &tot);
#pragma unroll
    for (int k = 0; k < 16; ++k) hist[16 * t + k] = (unsigned short)(base + loc[k]);
    __syncthreads();
    for (int i = b0; i < b1; ++i) {
      const int p = A[i];
      unsigned short& o = hist[((idof(p) >> shift) & 15) * SEG_THREADS + t];
      Bf[o] = p;
      ++o;
    }
    __syncthreads();
    int* tmp = A;
    A = Bf;
    Bf = tmp;
  }
  // segments: a new one starts where the id changes
  int nf = 0;
  for (int i = b0; i < b1; ++i) nf += (i == 0 || idof(A[i]) != idof(A[i - 1])) ? 1 : 0;
  int nu;
  int u = seg_excl_scan(nf, sh, &nu);
  for (int i = b0; i < b1; ++i) {
    const int id = idof(A[i]);
    J.pos[i] = J.pos_base + A[i];
    if (i == 0 || id != idof(A[i - 1])) {
      J.off[u] = i;
      J.uq[u] = id;
      ++u;
    }
  }
  if (t == 0) {
    J.off[nu] = n;
    *J.nrows = nu;
  }
}

// dense[ids[u]][:] = rows[u][:]   (compact embedding grads -> dense, for DP all-reduce)
__global__ void scatter_rows_kernel(const float* __restrict__ rows, int E, const int* __restrict__ ids, int n,
                                    float* __restrict__ dense) {
  int u = blockIdx.x;
  if (u >= n) return;
  for (int e = threadIdx.x; e < E; e += blockDim.x) dense[(long long)ids[u] * E + e] = rows[(long long)u * E + e];
}

// ---------------------------------------------------------------------------
// elementwise
// ---------------------------------------------------------------------------
template <typename T>
__global__ void add2_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ o, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    o[i] = from_f<T>(to_f<T>(a[i]) + to_f<T>(b[i]));
}

template <typename TS, typename TD>
__global__ void copy2d_kernel(const TS* __restrict__ s, long long lds, TD* __restrict__ d, long long ldd, int rows,
                              int cols) {
  // 8 elements per thread when rows are 8-aligned (16-byte bf16 / 32-byte fp32 accesses)
  if ((cols & 7) == 0 && (lds & 7) == 0 && (ldd & 7) == 0 && (((uintptr_t)s | (uintptr_t)d) & 31) == 0) {
    const long long n8 = (long long)rows * (cols >> 3);
    const int c8 = cols >> 3;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
      const long long r = i / c8, c = (i % c8) * 8;
      const TS* sp = s + r * lds + c;
      TD* dp = d + r * ldd + c;
      float f[8];
      if constexpr (sizeof(TS) == 2) {
        const uint4 q = *(const uint4*)sp;
        const bf16* b = (const bf16*)&q;
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __bfloat162float(b[j]);
      } else {
        const float4 a = *(const float4*)sp, b = *((const float4*)sp + 1);
        f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
      }
      if constexpr (sizeof(TD) == 2) {
        __align__(16) bf16 o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = __float2bfloat16_rn(f[j]);
        *(uint4*)dp = *(const uint4*)o;
      } else {
        *(float4*)dp = make_float4(f[0], f[1], f[2], f[3]);
        *((float4*)dp + 1) = make_float4(f[4], f[5], f[6], f[7]);
      }
    }
    return;
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)rows * cols;
       i += (long long)gridDim.x * blockDim.x) {
    long long r = i / cols, c = i % cols;
    d[r * ldd + c] = from_f<TD>(to_f<TS>(s[r * lds + c]));
  }
}

__global__ void fill_kernel(float* p, long long n, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void to_bf16_kernel(const float* __restrict__ s, bf16* __restrict__ d, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = __float2bfloat16_rn(s[i]);
}

// ---------------------------------------------------------------------------
// PCG64 (numpy's default bit generator: 128-bit LCG + XSL-RR output) with
// O(log n) jump-ahead, so every dropout element regenerates the exact double
// numpy's Generator.random() draws for it (reference layers.py:283).
// ---------------------------------------------------------------------------
typedef unsigned __int128 u128;
struct Pcg {
  unsigned long long state_hi, state_lo, inc_hi, inc_lo;
};
// The per-step values the kernels of a train step read from device memory
// (written by set_scalars_kernel at the start of each step), so that one
// captured CUDA graph serves every batch of a shape bucket.
struct StepScalars {
  Pcg pcg;              // generator state before the step's first draw
  double lr, clip;      // SGD rate, global-norm clip (NaN / < 0: none)
  float eps, inv_ntok;  // label smoothing, 1 / target tokens
  int nrows[2];         // unique embedding rows of the batch per table
};
__global__ void set_scalars_kernel(StepScalars v, StepScalars* __restrict__ d) { *d = v; }
// timeline mode: hold the stream while the host enqueues the whole step, so the
// per-launch events measure device time, not the host's launch rate
__global__ void hold_kernel(unsigned long long ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (t - t0 >= ns) break;
    __nanosleep(1000);
  }
}
CMT_D u128 pcg_mult() {
  return ((u128)0x2360ed051fc65da4ULL << 64) | (u128)0x4385df649fccf645ULL;
}
CMT_D u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}
CMT_D unsigned long long pcg_out(u128 s) {
  unsigned long long hi = (unsigned long long)(s >> 64), lo = (unsigned long long)s;
  unsigned rot = (unsigned)(s >> 122);
  unsigned long long x = hi ^ lo;
  return (x >> rot) | (x << ((64 - rot) & 63));
}

// Jump-ahead table of the PCG64 LCG for one stream increment: advancing by
// 2^i steps is s -> m[i] s + p[i].  Built once per increment (one thread), it
// turns each thread's jump to its first draw into one 128-bit multiply-add per
// set bit of the offset instead of a square-and-multiply loop.
struct PcgJump {
  u128 m[64], p[64];
};
__global__ void pcg_jump_table_kernel(PcgJump* t, unsigned long long inc_hi, unsigned long long inc_lo) {
  u128 m = pcg_mult(), pl = ((u128)inc_hi << 64) | inc_lo;
  for (int i = 0; i < 64; ++i) {
    t->m[i] = m;
    t->p[i] = pl;
    pl = (m + 1) * pl;
    m = m * m;
  }
}
CMT_D u128 pcg_jump(const PcgJump* __restrict__ t, u128 s, unsigned long long delta) {
  while (delta) {
    const int i = __ffsll((long long)delta) - 1;
    s = t->m[i] * s + t->p[i];
    delta &= delta - 1;
  }
  return s;
}

// Dropout site y = x * keep/(1-p) of shape (H, N) in the reference's C order:
// element (h, n) is draw (base + h*N + n) of numpy's Generator.random.
// keep  <=>  (r >> 11) * 2^-53 >= p  <=>  (r >> 11) >= ceil(p * 2^53): the
// reference's double comparison done exactly in integers (p * 2^53 is exact).
inline unsigned long long dropout_threshold(double p) { return (unsigned long long)std::ceil(p * 9007199254740992.0); }
// The PCG64 jump-ahead starts each thread's run of draws; the LCG step is written in 64-bit halves
// against the constant PCG64 multiplier (one umulhi, three low products, one
// carry), the keep test on the state halves directly, and the element index
// advanced incrementally: about half the instructions per draw.
#ifndef CMT_DROP_DPT
#define CMT_DROP_DPT 64
#endif
constexpr int DROP4_DPT = CMT_DROP_DPT;  // draws per thread: one jump-ahead amortised over them
template <typename TI, typename TO>
__global__ void dropout_fwd_kernel4(const TI* __restrict__ x, TO* __restrict__ y, uint8_t* __restrict__ keep, int N,
                                    int H, const Pcg* __restrict__ pcgp, const PcgJump* __restrict__ jt,
                                    unsigned long long base, unsigned long long thr, float scale,
                                    const TI* __restrict__ x2 = nullptr) {
  const int h = blockIdx.x * 32 + threadIdx.x;
  const int n0 = (blockIdx.y * blockDim.y + threadIdx.y) * DROP4_DPT;
  if (h >= H || n0 >= N) return;
  const Pcg pcg = *pcgp;
  const u128 s0 = pcg_jump(jt, ((u128)pcg.state_hi << 64) | pcg.state_lo, base + (unsigned long long)h * N + n0);
  unsigned long long sh = (unsigned long long)(s0 >> 64), sl = (unsigned long long)s0;
  const unsigned long long MH = 0x2360ed051fc65da4ULL, ML = 0x4385df649fccf645ULL;
  const unsigned long long ih = pcg.inc_hi, il = pcg.inc_lo;
  const int nend = min(N, n0 + DROP4_DPT);
  long long i = (long long)n0 * H + h;
#pragma unroll 4
  for (int n = n0; n < nend; ++n, i += H) {
    const unsigned long long lo = sl * ML;
    const unsigned long long hi = __umul64hi(sl, ML) + sl * MH + sh * ML;
    sl = lo + il;
    sh = hi + ih + (sl < lo ? 1ull : 0ull);
    const unsigned rot = (unsigned)(sh >> 58);
    const unsigned long long xr = sh ^ sl;
    const unsigned long long r = (xr >> rot) | (xr << ((64 - rot) & 63));
    const bool k = (r >> 11) >= thr;
    keep[i] = k;
    // x2: the input is x + x2 rounded to TI, exactly what add2_kernel stores
    // (the bidirectional sum of encoder layer 1, layers.py:162-180)
    const float xv = x2 ? to_f<TI>(from_f<TI>(to_f<TI>(x[i]) + to_f<TI>(x2[i]))) : to_f<TI>(x[i]);
    y[i] = from_f<TO>(k ? xv * scale : xv * 0.f);
  }
}

// Dropout masks ahead of their sites: the keep bytes of a site depend only
// on the generator state and the site's draw base, not on the data, so the
// step generates them on the SMs a running recurrent scan leaves idle (a few
// persistent CTAs, one per SM) and the site itself becomes a memory-bound
// apply.  Same draws and the same keep test as dropout_fwd_kernel4.
constexpr int DMASK_THREADS = 1024;
constexpr int DMASK_SMEM = 120 * 1024;  // one CTA per SM: a scan CTA never shares the SM
__global__ void __launch_bounds__(DMASK_THREADS, 1)
    dropout_mask_kernel(uint8_t* __restrict__ keep, int N, int H, const Pcg* __restrict__ pcgp,
                        const PcgJump* __restrict__ jt, unsigned long long base, unsigned long long thr) {
  const Pcg pcg = *pcgp;
  const unsigned long long MH = 0x2360ed051fc65da4ULL, ML = 0x4385df649fccf645ULL;
  const unsigned long long ih = pcg.inc_hi, il = pcg.inc_lo;
  const int chunks = (N + DROP4_DPT - 1) / DROP4_DPT;
  const long long items = (long long)chunks * H;  // item w: unit h = w % H, draws n0 = (w / H) * DPT
  for (long long w = blockIdx.x * (long long)DMASK_THREADS + threadIdx.x; w < items;
       w += (long long)gridDim.x * DMASK_THREADS) {
    const int h = (int)(w % H);
    const int n0 = (int)(w / H) * DROP4_DPT;
    const u128 s0 = pcg_jump(jt, ((u128)pcg.state_hi << 64) | pcg.state_lo, base + (unsigned long long)h * N + n0);
    unsigned long long sh = (unsigned long long)(s0 >> 64), sl = (unsigned long long)s0;
    const int nend = min(N, n0 + DROP4_DPT);
    long long i = (long long)n0 * H + h;
#pragma unroll 4
    for (int n = n0; n < nend; ++n, i += H) {
      const unsigned long long lo = sl * ML;
      const unsigned long long hi = __umul64hi(sl, ML) + sl * MH + sh * ML;
      sl = lo + il;
      sh = hi + ih + (sl < lo ? 1ull : 0ull);
      const unsigned rot = (unsigned)(sh >> 58);
      const unsigned long long xr = sh ^ sl;
      const unsigned long long r = (xr >> rot) | (xr << ((64 - rot) & 63));
      keep[i] = (r >> 11) >= thr;
    }
  }
}
// y = x * keep / (1 - p) with the masks above (x + x2 first for the
// bidirectional sum feeding enc.l2, rounded to TI as add2_kernel stores it)
template <typename TI, typename TO>
__global__ void dropout_apply_kernel(const TI* __restrict__ x, const TI* __restrict__ x2,
                                     const uint8_t* __restrict__ keep, TO* __restrict__ y, long long n, float scale) {
  const long long n8 = n >> 3;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n8; v += (long long)gridDim.x * blockDim.x) {
    const uint2 kb = ((const uint2*)keep)[v];
    const uint8_t* k8 = (const uint8_t*)&kb;
    float xv[8];
    if constexpr (sizeof(TI) == 2) {
      const uint4 a = ((const uint4*)x)[v];
      const TI* a8 = (const TI*)&a;
      if (x2) {
        const uint4 b = ((const uint4*)x2)[v];
        const TI* b8 = (const TI*)&b;
#pragma unroll
        for (int j = 0; j < 8; ++j) xv[j] = to_f<TI>(from_f<TI>(to_f<TI>(a8[j]) + to_f<TI>(b8[j])));
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) xv[j] = to_f<TI>(a8[j]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float a = to_f<TI>(x[v * 8 + j]);
        xv[j] = x2 ? to_f<TI>(from_f<TI>(a + to_f<TI>(x2[v * 8 + j]))) : a;
      }
    }
    TO o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = from_f<TO>(k8[j] ? xv[j] * scale : xv[j] * 0.f);
    if constexpr (sizeof(TO) == 2) {
      ((uint4*)y)[v] = *(const uint4*)o;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) y[v * 8 + j] = o[j];
    }
  }
  // tail (n % 8)
  for (long long i = n8 * 8 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float a = to_f<TI>(x[i]);
    if (x2) a = to_f<TI>(from_f<TI>(a + to_f<TI>(x2[i])));
    y[i] = from_f<TO>(keep[i] ? a * scale : a * 0.f);
  }
}

// ---------------------------------------------------------------------------
// Luong "general" attention, one CTA per sentence b (attention.py:46-84,
// layers.py:183-215).  Hs rows n = s*B+b, queries n = t*B+b.
// ---------------------------------------------------------------------------
constexpr int ATT_THREADS = 256;
constexpr int ATT_MAXP = 64;  // register tile: S*T <= 64*256
constexpr int ATT_HC = 32;

inline size_t attn_fwd_smem(int S, int T) { return sizeof(float) * ((size_t)T * (S + 1) + (size_t)(S + T) * (ATT_HC + 1)); }
inline size_t attn_bwd_smem(int S, int T) {
  return sizeof(float) * (2 * (size_t)T * (S + 1) + (size_t)(S + 2 * T) * (ATT_HC + 1));
}

// sc[t][s] = sum_h P[t][h] * Q[s][h] over all H (P rows t*B+b, Q rows s*B+b)
template <typename TP, typename TQ>
CMT_D void att_scores(const TP* P, long long ldp, const TQ* Q, long long ldq, int S, int T, int B, int H, int b,
                      float* sc, float* tP, float* tQ) {
  const int tid = threadIdx.x;
  float acc[ATT_MAXP];
#pragma unroll
  for (int r = 0; r < ATT_MAXP; ++r) acc[r] = 0.f;
  const int np = S * T;
  for (int h0 = 0; h0 < H; h0 += ATT_HC) {
    for (int i = tid; i < T * ATT_HC; i += ATT_THREADS) {
      int t = i / ATT_HC, hh = i % ATT_HC;
      tP[t * (ATT_HC + 1) + hh] = (h0 + hh < H) ? to_f<TP>(P[(long long)(t * B + b) * ldp + h0 + hh]) : 0.f;
    }
    for (int i = tid; i < S * ATT_HC; i += ATT_THREADS) {
      int s = i / ATT_HC, hh = i % ATT_HC;
      tQ[s * (ATT_HC + 1) + hh] = (h0 + hh < H) ? to_f<TQ>(Q[(long long)(s * B + b) * ldq + h0 + hh]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < ATT_MAXP; ++r) {
      int q = tid + r * ATT_THREADS;
      if (q < np) {
        int t = q / S, s = q % S;
        const float* pp = tP + t * (ATT_HC + 1);
        const float* qq = tQ + s * (ATT_HC + 1);
        float a = acc[r];
#pragma unroll
        for (int hh = 0; hh < ATT_HC; ++hh) a = fmaf(pp[hh], qq[hh], a);
        acc[r] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < ATT_MAXP; ++r) {
    int q = tid + r * ATT_THREADS;
    if (q < np) sc[(q / S) * (S + 1) + (q % S)] = acc[r];
  }
  __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(ATT_THREADS) attn_fwd_kernel(const T* __restrict__ Hs, const T* __restrict__ U,
                                                               const float* __restrict__ src_mask, int S, int Tq,
                                                               int B, int H, float* __restrict__ alpha,
                                                               T* __restrict__ ctx, long long ldctx,
                                                               int* __restrict__ status) {
  extern __shared__ float sm[];
  const int b = blockIdx.x;
  float* sc = sm;                                // [T][S+1]
  float* tP = sc + Tq * (S + 1);                 // [T][HC+1]
  float* tQ = tP + Tq * (ATT_HC + 1);            // [S][HC+1]
  att_scores(U, H, Hs, H, S, Tq, B, H, b, sc, tP, tQ);
  // masked column softmax over s (additive -1e9 as in layers.py:190/202)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = warp; t < Tq; t += ATT_THREADS / 32) {
    float* row = sc + t * (S + 1);
    float mx = -INFINITY;
    bool bad = false;
    for (int s = lane; s < S; s += 32) {
      float v = row[s] + (1.f - src_mask[s * B + b]) * -1e9f;
      bad |= !isfinite(v);
      row[s] = v;
      mx = fmaxf(mx, v);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int s = lane; s < S; s += 32) {
      float e = expf(row[s] - mx);
      row[s] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    float inv = 1.f / sum;
    for (int s = lane; s < S; s += 32) {
      float a = row[s] / sum;
      row[s] = a;
      alpha[((long long)b * Tq + t) * S + s] = a;
    }
    (void)inv;
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_SCORES);
  }
  __syncthreads();
  // context: ctx[t][h] = sum_s alpha[t][s] Hs[s][h]
  for (int h0 = 0; h0 < H; h0 += ATT_HC) {
    for (int i = threadIdx.x; i < S * ATT_HC; i += ATT_THREADS) {
      int s = i / ATT_HC, hh = i % ATT_HC;
      tQ[s * (ATT_HC + 1) + hh] = (h0 + hh < H) ? to_f<T>(Hs[(long long)(s * B + b) * H + h0 + hh]) : 0.f;
    }
    __syncthreads();
    const int hh = threadIdx.x & 31;
    for (int t = threadIdx.x >> 5; t < Tq; t += ATT_THREADS / 32) {
      const float* row = sc + t * (S + 1);
      float a = 0.f;
      for (int s = 0; s < S; ++s) a = fmaf(row[s], tQ[s * (ATT_HC + 1) + hh], a);
      if (h0 + hh < H) ctx[(long long)(t * B + b) * ldctx + h0 + hh] = from_f<T>(a);
    }
    __syncthreads();
  }
}

// backward: given dC (= dCst[:, :H], fp32), produce dHs (+=) and du (act).
template <typename T>
__global__ void __launch_bounds__(ATT_THREADS) attn_bwd_kernel(const T* __restrict__ Hs, const T* __restrict__ U,
                                                               const float* __restrict__ alpha,
                                                               const float* __restrict__ dC, long long lddc, int S,
                                                               int Tq, int B, int H, float* __restrict__ dHs,
                                                               T* __restrict__ dU) {
  extern __shared__ float sm[];
  const int b = blockIdx.x;
  float* da = sm;                         // [T][S+1]  d alpha -> d scores
  float* al = da + Tq * (S + 1);          // [T][S+1]  alpha
  float* tP = al + Tq * (S + 1);          // [T][HC+1]
  float* tQ = tP + Tq * (ATT_HC + 1);     // [S][HC+1]
  float* tR = tQ + S * (ATT_HC + 1);      // [T][HC+1]
  // d alpha[t][s] = sum_h dC[t][h] Hs[s][h]
  att_scores(dC, lddc, Hs, H, S, Tq, B, H, b, da, tP, tQ);
  for (int i = threadIdx.x; i < Tq * S; i += ATT_THREADS) {
    int t = i / S, s = i % S;
    al[t * (S + 1) + s] = alpha[((long long)b * Tq + t) * S + s];
  }
  __syncthreads();
  // d scores = p * (g - sum_s p g)   (layers.py:210-215)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = warp; t < Tq; t += ATT_THREADS / 32) {
    float* g = da + t * (S + 1);
    const float* p = al + t * (S + 1);
    float dot = 0.f;
    for (int s = lane; s < S; s += 32) dot += p[s] * g[s];
    dot = warp_sum(dot);
    for (int s = lane; s < S; s += 32) g[s] = p[s] * (g[s] - dot);
  }
  __syncthreads();
  const int hh = threadIdx.x & 31;
  for (int h0 = 0; h0 < H; h0 += ATT_HC) {
    for (int i = threadIdx.x; i < Tq * ATT_HC; i += ATT_THREADS) {
      int t = i / ATT_HC, c = i % ATT_HC;
      bool ok = h0 + c < H;
      tP[t * (ATT_HC + 1) + c] = ok ? dC[(long long)(t * B + b) * lddc + h0 + c] : 0.f;
      tR[t * (ATT_HC + 1) + c] = ok ? to_f<T>(U[(long long)(t * B + b) * H + h0 + c]) : 0.f;
    }
    for (int i = threadIdx.x; i < S * ATT_HC; i += ATT_THREADS) {
      int s = i / ATT_HC, c = i % ATT_HC;
      tQ[s * (ATT_HC + 1) + c] = (h0 + c < H) ? to_f<T>(Hs[(long long)(s * B + b) * H + h0 + c]) : 0.f;
    }
    __syncthreads();
    // dHs[s][h] += sum_t alpha[t][s] dC[t][h] + dscores[t][s] U[t][h]
    for (int s = threadIdx.x >> 5; s < S; s += ATT_THREADS / 32) {
      float a = 0.f;
      for (int t = 0; t < Tq; ++t)
        a = fmaf(al[t * (S + 1) + s], tP[t * (ATT_HC + 1) + hh], fmaf(da[t * (S + 1) + s], tR[t * (ATT_HC + 1) + hh], a));
      if (h0 + hh < H) dHs[(long long)(s * B + b) * H + h0 + hh] += a;
    }
    // du[t][h] = sum_s dscores[t][s] Hs[s][h]
    for (int t = threadIdx.x >> 5; t < Tq; t += ATT_THREADS / 32) {
      const float* g = da + t * (S + 1);
      float a = 0.f;
      for (int s = 0; s < S; ++s) a = fmaf(g[s], tQ[s * (ATT_HC + 1) + hh], a);
      if (h0 + hh < H) dU[(long long)(t * B + b) * H + h0 + hh] = from_f<T>(a);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Fused log-softmax + label-smoothed CE + gradient (+ tanh'), one CTA per
// token row of the [N_T][V] logits; the gradient overwrites the logits.
// loss_n = lse - (1-eps) y_gold - (eps/V) sum_v y_v            (training.py:111-113)
// d_v    = (e^{y_v-lse} - eps/V - (1-eps)[v=gold]) m_n / ntok  (training.py:116-119)
// dpre_v = d_v (1 - y_v^2) when the output tanh is on           (layers.py:136-138)
// ---------------------------------------------------------------------------
constexpr int CE_THREADS = 512;
template <typename T>
__global__ void __launch_bounds__(CE_THREADS) ce_kernel(T* __restrict__ Y, int V, const int* __restrict__ tgt,
                                                        const float* __restrict__ tmask,
                                                        const StepScalars* __restrict__ sc, int tanh_on,
                                                        float* __restrict__ losstok, int* __restrict__ status) {
  const float eps = sc->eps, inv_ntok = sc->inv_ntok;
  __shared__ float red_m[CE_THREADS / 32], red_s[CE_THREADS / 32], red_y[CE_THREADS / 32];
  __shared__ float bc[2];
  const long long n = blockIdx.x;
  T* row = Y + n * V;
  float mx = -INFINITY, se = 0.f, sy = 0.f;
  bool bad = false;
  for (int v = threadIdx.x; v < V; v += CE_THREADS) {
    float y = to_f<T>(row[v]);
    bad |= !isfinite(y);
    sy += y;
    if (y > mx) {
      se = se * expf(mx - y) + 1.f;
      mx = y;
    } else {
      se += expf(y - mx);
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float wm = warp_max(mx);
  se = (mx == -INFINITY) ? 0.f : se * expf(mx - wm);
  se = warp_sum(se);
  sy = warp_sum(sy);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_LOGITS);
  if (lane == 0) { red_m[warp] = wm; red_s[warp] = se; red_y[warp] = sy; }
  __syncthreads();
  if (warp == 0) {
    float m2 = lane < CE_THREADS / 32 ? red_m[lane] : -INFINITY;
    float s2 = lane < CE_THREADS / 32 ? red_s[lane] : 0.f;
    float y2 = lane < CE_THREADS / 32 ? red_y[lane] : 0.f;
    float gm = warp_max(m2);
    s2 = (m2 == -INFINITY) ? 0.f : s2 * expf(m2 - gm);
    s2 = warp_sum(s2);
    y2 = warp_sum(y2);
    if (lane == 0) {
      float lse = gm + logf(s2);
      int g = tgt[n];
      float gold = to_f<T>(row[g]);
      float per = lse - (1.f - eps) * gold - (eps / (float)V) * y2;
      // reference per_token = -((1-eps) lp_gold + (eps/V) sum lp)  with lp = y - lse
      float m = tmask[n];
      losstok[n] = per * m;
      if (!isfinite(per)) atomicOr(status, ST_LOSS);
      bc[0] = lse;
      bc[1] = m * inv_ntok;
    }
  }
  __syncthreads();
  const float lse = bc[0], w = bc[1];
  const int g = tgt[n];
  const float eV = eps / (float)V;
  for (int v = threadIdx.x; v < V; v += CE_THREADS) {
    float y = to_f<T>(row[v]);
    float d = expf(y - lse) - eV - (v == g ? (1.f - eps) : 0.f);
    d *= w;
    if (tanh_on) d *= (1.f - y * y);
    row[v] = from_f<T>(d);
  }
}

// deterministic sum of a float vector into a double (single CTA)
__global__ void sum_to_double_kernel(const float* __restrict__ x, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double a = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a += (double)x[i];
  a = warp_sumd(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sumd(v);
    if (threadIdx.x == 0) *out = v;
  }
}

// ---------------------------------------------------------------------------
// Column sums (bias grads: layers.py:72-73, 391): partial over row chunks,
// then a fixed-order combine -> deterministic.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Fused CE over bf16 logits (production path; rows 16-byte aligned), same math
// as ce_kernel (training.py:96-120, tensor.py:146-151).
// ---------------------------------------------------------------------------
constexpr float kLog2e = 1.4426950408889634f;
CMT_D float ex2f(float x) {  // 2^x (MUFU.EX2)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Two-pass fused CE (ce2 = 2, default): both passes run at full occupancy
// with no shared-memory column accumulators.
// Pass 1, one CTA per token row: log-sum-exp, smoothed per-token loss and the
// row's (lse*log2e, mask/ntok) for pass 2 (training.py:96-120, tensor.py:146-151).
constexpr int CES_THREADS = 512;
#ifndef CMT_CES_MINB
#define CMT_CES_MINB 1  // (3 CTAs per SM forces spills: 147.5 -> 151.6 us)
#endif
__global__ void __launch_bounds__(CES_THREADS, CMT_CES_MINB) ce_stats_kernel(const bf16* __restrict__ Y, int V,
                                                               const int* __restrict__ tgt,
                                                               const float* __restrict__ tmask,
                                                               const StepScalars* __restrict__ sc, int tanh_on,
                                                               float* __restrict__ losstok,
                                                               int* __restrict__ status, float2* __restrict__ rowst) {
  const float eps = sc->eps, inv_ntok = sc->inv_ntok;
  __shared__ float red_m[CES_THREADS / 32], red_s[CES_THREADS / 32], red_y[CES_THREADS / 32];
  const int n = blockIdx.x;
  const int nv = V >> 3;
  const uint4* row = (const uint4*)(Y + (long long)n * V);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float mx = tanh_on ? 0.f : -INFINITY, se = 0.f, sy = 0.f;
  bool bad = false;
  for (int i0 = threadIdx.x; i0 < nv; i0 += 4 * CES_THREADS) {
    uint4 qv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * CES_THREADS;
      qv[u] = i < nv ? __ldg(row + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i0 + u * CES_THREADS >= nv) break;
      const bf16* e = (const bf16*)&qv[u];
      float y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        y[j] = __bfloat162float(e[j]);
        sy += y[j];
      }
      if (tanh_on) {  // |y| <= 1: no max shift; non-finite logits surface in the row sum
#pragma unroll
        for (int j = 0; j < 8; ++j) se += ex2f(y[j] * kLog2e);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) bad |= !isfinite(y[j]);
        float lm = y[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) lm = fmaxf(lm, y[j]);
        if (lm > mx) {
          se = (mx == -INFINITY) ? 0.f : se * __expf(mx - lm);
          mx = lm;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) se += __expf(y[j] - mx);
      }
    }
  }
  const float wm = warp_max(mx);
  se = (mx == -INFINITY) ? 0.f : se * __expf(mx - wm);
  se = warp_sum(se);
  sy = warp_sum(sy);
  if (tanh_on) bad = !isfinite(sy);
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_LOGITS);
  if (lane == 0) { red_m[warp] = wm; red_s[warp] = se; red_y[warp] = sy; }
  __syncthreads();
  if (warp == 0) {
    const float m2 = lane < CES_THREADS / 32 ? red_m[lane] : -INFINITY;
    float s2 = lane < CES_THREADS / 32 ? red_s[lane] : 0.f;
    float y2 = lane < CES_THREADS / 32 ? red_y[lane] : 0.f;
    const float gm = warp_max(m2);
    s2 = (m2 == -INFINITY) ? 0.f : s2 * __expf(m2 - gm);
    s2 = warp_sum(s2);
    y2 = warp_sum(y2);
    if (lane == 0) {
      const float lse = gm + logf(s2);
      const float gold = __bfloat162float(Y[(long long)n * V + tgt[n]]);
      const float per = lse - (1.f - eps) * gold - (eps / (float)V) * y2;
      const float m = tmask[n];
      losstok[n] = per * m;
      if (!isfinite(per)) atomicOr(status, ST_LOSS);
      rowst[n] = make_float2(lse * kLog2e, m * inv_ntok);
    }
  }
}
// Pass 2: CTA = (2048-column slice, chunk of CEG_ROWS rows); a thread owns 8
// adjacent columns: it rewrites Y in place with the gradient
// d = (p - eps/V - (1-eps)[v=gold]) m/ntok (* (1 - y^2) under the output tanh)
// and keeps the 8 column sums (the bias grad, layers.py:72-73) in registers;
// part[chunk][v] is reduced by colsum_final_kernel in chunk order.
constexpr int CEG_THREADS = 256;
#ifndef CMT_CEG_MINB
#define CMT_CEG_MINB 6  // 48 warps per SM: 233.5 -> 221.2 us per c3 step
#endif
constexpr int CEG_COLS = 8 * CEG_THREADS;
constexpr int CEG_ROWS = 64;
__global__ void __launch_bounds__(CEG_THREADS, CMT_CEG_MINB) ce_grad_kernel(bf16* __restrict__ Y, int V, int rows,
                                                              const int* __restrict__ tgt,
                                                              const float2* __restrict__ rowst,
                                                              const StepScalars* __restrict__ sc, int tanh_on,
                                                              float* __restrict__ part) {
  const float eps = sc->eps;
  const int c = blockIdx.x * CEG_COLS + threadIdx.x * 8;
  // row chunks from the last: ce_stats_kernel has just read the logits in row
  // order, so the last rows are still in L2
  const int chunk = gridDim.y - 1 - blockIdx.y;
  const int r0 = chunk * CEG_ROWS, r1 = min(rows, r0 + CEG_ROWS);
  if (c >= V) return;
  const float eV = eps / (float)V;
  float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int rb = r0; rb < r1; rb += 4) {
    uint4 qv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      qv[u] = rb + u < r1 ? __ldcs((const uint4*)(Y + (long long)(rb + u) * V + c)) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = rb + u;
      if (r >= r1) break;
      const float2 st = __ldg(rowst + r);  // (lse * log2e, m / ntok)
      const int gj = __ldg(tgt + r) - c;    // the gold column falls in this vector iff 0 <= gj < 8
      const float ewv = eV * st.y, gw = (1.f - eps) * st.y;
      const bf16* e = (const bf16*)&qv[u];
      __align__(16) bf16 o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float y = __bfloat162float(e[j]);
        float d = fmaf(ex2f(fmaf(y, kLog2e, -st.x)), st.y, -ewv);
        if (j == gj) d -= gw;
        if (tanh_on) d *= fmaf(-y, y, 1.f);
        o[j] = __float2bfloat16_rn(d);
        cs[j] += d;
      }
      __stcs((uint4*)(Y + (long long)r * V + c), *(const uint4*)o);
    }
  }
  float4* pp = (float4*)(part + (long long)chunk * V + c);
  pp[0] = make_float4(cs[0], cs[1], cs[2], cs[3]);
  pp[1] = make_float4(cs[4], cs[5], cs[6], cs[7]);
}

template <typename T>
__global__ void colsum_partial_kernel(const T* __restrict__ D, long long ld, int rows, int cols, int rows_per,
                                      float* __restrict__ part) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  int r0 = blockIdx.y * rows_per, r1 = min(rows, r0 + rows_per);
  // 8 rows in flight per iteration (independent partial sums, fixed order)
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  int r = r0;
  for (; r + 8 <= r1; r += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] += to_f<T>(D[(long long)(r + k) * ld + c]);
  }
  for (; r < r1; ++r) a[0] += to_f<T>(D[(long long)r * ld + c]);
  part[(long long)blockIdx.y * cols + c] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}
// bf16 rows: a CTA covers 256 columns (threadIdx.x: 8 columns via 16-byte
// loads, a warp reads 512 contiguous bytes of a row) and 8 row lanes
// (threadIdx.y: rows r0 + y, r0 + y + 8, ...; 2 rows in flight); the 8 lanes'
// sums are combined in shared memory in lane order, so the partial of a chunk
// is deterministic.
// The last CTA of a column block to finish (a self-resetting ticket per column
// block) adds the chunks' partials in chunk order and writes out[col]: one
// launch, deterministic.
__global__ void __launch_bounds__(256) colsum_partial_v8_kernel(const bf16* __restrict__ D, long long ld, int rows,
                                                                int cols, int rows_per, float* __restrict__ part,
                                                                unsigned* __restrict__ ticket, float* __restrict__ out) {
  __shared__ float red[8][256 + 4];
  const int cx = threadIdx.x * 8, c = blockIdx.x * 256 + cx;
  const int r0 = blockIdx.y * rows_per, r1 = min(rows, r0 + rows_per);
  float a[2][8];
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[k][j] = 0.f;
  if (c < cols) {
    int r = r0 + threadIdx.y;
    for (; r + 8 < r1; r += 16) {
      const uint4 q0 = __ldcs((const uint4*)(D + (long long)r * ld + c));
      const uint4 q1 = __ldcs((const uint4*)(D + (long long)(r + 8) * ld + c));
      const bf16* e0 = (const bf16*)&q0;
      const bf16* e1 = (const bf16*)&q1;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a[0][j] += __bfloat162float(e0[j]);
        a[1][j] += __bfloat162float(e1[j]);
      }
    }
    if (r < r1) {
      const uint4 q0 = __ldcs((const uint4*)(D + (long long)r * ld + c));
      const bf16* e0 = (const bf16*)&q0;
#pragma unroll
      for (int j = 0; j < 8; ++j) a[0][j] += __bfloat162float(e0[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[threadIdx.y][cx + j] = a[0][j] + a[1][j];
  __syncthreads();
  // 256 threads, one column each: sum the 8 row lanes in order
  const int t = threadIdx.y * 32 + threadIdx.x, col = blockIdx.x * 256 + t;
  if (col < cols) {
    float o = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) o += red[y][t];
    part[(long long)blockIdx.y * cols + col] = o;
  }
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (t == 0) last = atomicAdd(ticket + blockIdx.x, 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (col < cols) {
    float a = 0.f;
    for (int k = 0; k < (int)gridDim.y; ++k) a += __ldcg(part + (long long)k * cols + col);
    out[col] = a;
  }
  if (t == 0) ticket[blockIdx.x] = 0;  // ready for the next launch
}
__global__ void colsum_final_kernel(const float* __restrict__ part, int chunks, int cols, float* __restrict__ out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float a = 0.f;
  for (int k = 0; k < chunks; ++k) a += part[(long long)k * cols + c];
  out[c] = a;
}

// ---------------------------------------------------------------------------
// Global-norm clip + SGD (training.py:123-142)
// ---------------------------------------------------------------------------
constexpr int NORM_BLOCKS = 592;  // 4 x 148 SMs
// Gate (de)interleave for parameter upload / download: the reference block
// w_q (rows, H) is column 4j+q of the engine's [rows][4H] layer matrix.
// to_inter: plain -> interleaved (upload); else interleaved -> plain (download).
__global__ void gate_copy_kernel(float* __restrict__ inter, float* __restrict__ plain, long long rows, int H,
                                 int q, int to_inter) {
  const long long n = rows * H;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / H, j = i - r * H;
    float* d = inter + r * 4LL * H + 4 * j + q;
    if (to_inter) *d = plain[i];
    else plain[i] = *d;
  }
}

// lanes: 4-bit gate mask; element i (from g) counts iff bit (i & 3) is set
// (15 = every element; in a gate-interleaved LSTM region i & 3 is the gate)
// nrows_d (optional): n = *nrows_d * rowlen, the embedding rows of the step
__global__ void sumsq_partial_kernel(const float* __restrict__ g, long long n, double* __restrict__ part,
                                     int lanes, const int* __restrict__ nrows_d = nullptr, int rowlen = 0) {
  if (nrows_d) n = (long long)*nrows_d * rowlen;
  __shared__ double red[32];
  float a = 0.f;
  double ad = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool l0 = lanes & 1, l1 = lanes & 2, l2 = lanes & 4, l3 = lanes & 8;
  int cnt = 0;
  if ((((uintptr_t)g) & 15) == 0) {
    const long long n4 = n >> 2;
    const float4* g4 = (const float4*)g;
    long long i = tid;
    for (; i + 3 * stride < n4; i += 4 * stride) {  // 4 independent 16-byte loads in flight
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(g4 + i + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a = fmaf(l0 ? v[u].x : 0.f, l0 ? v[u].x : 0.f, a);
        a = fmaf(l1 ? v[u].y : 0.f, l1 ? v[u].y : 0.f, a);
        a = fmaf(l2 ? v[u].z : 0.f, l2 ? v[u].z : 0.f, a);
        a = fmaf(l3 ? v[u].w : 0.f, l3 ? v[u].w : 0.f, a);
      }
      if (++cnt == 16) { ad += a; a = 0.f; cnt = 0; }
    }
    for (; i < n4; i += stride) {
      const float4 v = g4[i];
      a = fmaf(l0 ? v.x : 0.f, l0 ? v.x : 0.f, a);
      a = fmaf(l1 ? v.y : 0.f, l1 ? v.y : 0.f, a);
      a = fmaf(l2 ? v.z : 0.f, l2 ? v.z : 0.f, a);
      a = fmaf(l3 ? v.w : 0.f, l3 ? v.w : 0.f, a);
    }
    for (long long j = 4 * n4 + tid; j < n; j += stride)
      if ((lanes >> (j & 3)) & 1) a = fmaf(g[j], g[j], a);
  } else {
    for (long long i = tid; i < n; i += stride) {
      const float v = ((lanes >> (i & 3)) & 1) ? g[i] : 0.f;
      a = fmaf(v, v, a);
      if (++cnt == 256) { ad += a; a = 0.f; cnt = 0; }
    }
  }
  ad += a;
  ad = warp_sumd(ad);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ad;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sumd(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

// scal[0] = sum of squares, scal[1] = norm; s32 = fp32(lr * scale)
__global__ void clip_scale_kernel(const double* __restrict__ part, int nparts, const StepScalars* __restrict__ sc,
                                  double* __restrict__ scal, float* __restrict__ s32, int* __restrict__ status) {
  const double lr = sc->lr, clip = sc->clip;
  // fixed-shape reduction (strided per-thread sums, then a fixed tree), so the
  // norm is deterministic; launched with CLIP_THREADS threads
  __shared__ double red[32];
  double sq = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) sq += part[i];
  sq = warp_sumd(sq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  sq = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
  sq = warp_sumd(sq);
  if (threadIdx.x != 0) return;
  double norm = sqrt(sq);
  scal[0] = sq;
  scal[1] = norm;
  if (!isfinite(norm)) atomicOr(status, ST_NORM);
  double scale = 1.0;
  if (clip >= 0.0 && norm > clip) scale = clip / norm;  // clip < 0 or NaN: None
  *s32 = (float)(lr * scale);
}
constexpr int CLIP_THREADS = 512;

constexpr int ST_ABORT = ST_SCORES | ST_LOGITS | ST_LOSS | ST_NORM | ST_HANG;

// Data parallel: the ranks' status words are combined flag by flag.  A rank's
// word is spread into one int per flag, the ints are max-reduced over ranks
// (ncclMax) and the word is rebuilt, so k ranks raising the same flag give that
// flag, never a carry into another one (status_combine is the host statement of
// the same rule, exported for the CPU test).
constexpr int ST_NFLAGS = 5;
CMT_HD int status_spread(int s, int i) { return (s >> i) & 1; }
CMT_HD int status_rebuild(const int* f) {
  int s = 0;
  for (int i = 0; i < ST_NFLAGS; ++i) s |= f[i] ? (1 << i) : 0;
  return s;
}
inline int status_combine(const int* words, int n) {  // = spread, max over ranks, rebuild
  int f[ST_NFLAGS] = {0, 0, 0, 0, 0};
  for (int r = 0; r < n; ++r)
    for (int i = 0; i < ST_NFLAGS; ++i) f[i] = f[i] > status_spread(words[r], i) ? f[i] : status_spread(words[r], i);
  return status_rebuild(f);
}
__global__ void status_spread_kernel(const int* __restrict__ status, int* __restrict__ f) {
  if (threadIdx.x < ST_NFLAGS) f[threadIdx.x] = status_spread(*status, threadIdx.x);
}
__global__ void status_gather_kernel(const int* __restrict__ f, int* __restrict__ status) {
  if (threadIdx.x == 0) *status = status_rebuild(f);
}

// w -= fp32(lr * scale) * g over the elements whose gate bit (i & 3) is set in lanes
__global__ void sgd_dense_kernel(float* __restrict__ w, const float* __restrict__ g, bf16* __restrict__ shadow,
                                 long long n, const float* __restrict__ s32, const int* __restrict__ status,
                                 int lanes) {
  if (*status & ST_ABORT) return;
  const float s = *s32;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool l0 = lanes & 1, l1 = lanes & 2, l2 = lanes & 4, l3 = lanes & 8;
  // 16-byte vectors over the (256-byte aligned) arena, scalar tail
  const long long n4 = n >> 2;
  float4* w4 = (float4*)w;
  const float4* g4 = (const float4*)g;
  for (long long i0 = tid; i0 < n4; i0 += stride) {
    const long long i = n4 - 1 - i0;  // from the end: the norm pass has just read it (L2)
    const float4 wv = w4[i], gv = __ldcs(g4 + i);
    float4 nw;
    nw.x = l0 ? __fsub_rn(wv.x, __fmul_rn(s, gv.x)) : wv.x;
    nw.y = l1 ? __fsub_rn(wv.y, __fmul_rn(s, gv.y)) : wv.y;
    nw.z = l2 ? __fsub_rn(wv.z, __fmul_rn(s, gv.z)) : wv.z;
    nw.w = l3 ? __fsub_rn(wv.w, __fmul_rn(s, gv.w)) : wv.w;
    w4[i] = nw;
    if (shadow) {
      __align__(8) bf16 b4[4] = {__float2bfloat16_rn(nw.x), __float2bfloat16_rn(nw.y), __float2bfloat16_rn(nw.z),
                                 __float2bfloat16_rn(nw.w)};
      *(uint2*)(shadow + 4 * i) = *(uint2*)b4;
    }
  }
  for (long long i = 4 * n4 + tid; i < n; i += stride) {
    if (!((lanes >> (i & 3)) & 1)) continue;
    float nw = __fsub_rn(w[i], __fmul_rn(s, g[i]));
    w[i] = nw;
    if (shadow) shadow[i] = __float2bfloat16_rn(nw);
  }
}

__global__ void sgd_rows_kernel(float* __restrict__ table, bf16* __restrict__ shadow, int E,
                                const int* __restrict__ ids, int nrows, const float* __restrict__ gc,
                                const float* __restrict__ s32, const int* __restrict__ status,
                                const int* __restrict__ nrows_d = nullptr) {
  if (*status & ST_ABORT) return;
  int u = blockIdx.x;
  if (nrows_d) nrows = *nrows_d;
  if (u >= nrows) return;
  const float s = *s32;
  long long r = (long long)ids[u] * E;
  if ((E & 3) == 0) {  // float4 rows (the arena and tables are 256-byte aligned)
    float4* tw = (float4*)(table + r);
    const float4* g4 = (const float4*)(gc + (long long)u * E);
    for (int e = threadIdx.x; e < (E >> 2); e += blockDim.x) {
      const float4 w = tw[e], gv = g4[e];
      float4 nw;
      nw.x = __fsub_rn(w.x, __fmul_rn(s, gv.x));
      nw.y = __fsub_rn(w.y, __fmul_rn(s, gv.y));
      nw.z = __fsub_rn(w.z, __fmul_rn(s, gv.z));
      nw.w = __fsub_rn(w.w, __fmul_rn(s, gv.w));
      tw[e] = nw;
      if (shadow) {
        __align__(8) bf16 b4[4] = {__float2bfloat16_rn(nw.x), __float2bfloat16_rn(nw.y), __float2bfloat16_rn(nw.z),
                                   __float2bfloat16_rn(nw.w)};
        *(uint2*)(shadow + r + 4 * e) = *(uint2*)b4;
      }
    }
    return;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float nw = __fsub_rn(table[r + e], __fmul_rn(s, gc[(long long)u * E + e]));
    table[r + e] = nw;
    if (shadow) shadow[r + e] = __float2bfloat16_rn(nw);
  }
}

}  // namespace cmt
