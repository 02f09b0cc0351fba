// Luong "general" attention core, register-tiled (attention.py:46-84, 139-173;
// layers.py:183-215).  One CTA per sentence b; Hs rows n = s*B+b (source
// positions), query rows n = t*B+b (decoder steps).  S, T <= 64: each of the
// 256 threads owns a 4x4 block of a 64x64 tile, so every shared-memory read
// feeds 4 FMAs (the previous kernels did one FMA per two reads).
//
//   forward : scores = U Hs^T (U = W_a^T H_t, the u of attention.py:166),
//             masked column softmax with the additive -1e9 (exact zeros),
//             C_s = alpha Hs                       -> alpha (fp32), ctx
//   backward: dalpha = dC Hs^T, dscores = alpha (dalpha - sum_s alpha dalpha),
//             dHs += alpha^T dC + dscores^T U,  dU = dscores Hs
// All arithmetic is fp32; E is the activation storage type (bf16 / fp32).
#pragma once
#include "kernels.cuh"

namespace cmt {
namespace att {
constexpr int THREADS = 256;
constexpr int P = 64;       // padded S / T
constexpr int LD = P + 4;   // smem row stride (floats): float4-aligned rows
constexpr int KC = 32;      // h-chunk of the score products
constexpr int HC = 64;      // h-chunk of the context / gradient products

// dst[k][r] = src row r (global row r*B+b), columns k0..k0+KC-1 (transposed), zero padded
template <typename E>
CMT_D void load_t(float* dst, const E* src, long long ld, int rows, int B, int b, int k0, int K) {
  constexpr int VEC = 16 / sizeof(E);
  constexpr int SEGS = KC / VEC;
  for (int i = threadIdx.x; i < P * SEGS; i += THREADS) {
    const int r = i / SEGS, sg = i % SEGS;
    const int k = k0 + sg * VEC;
    float v[VEC];
    const E* p = src + ((long long)r * B + b) * ld + k;
    if (r < rows && k + VEC <= K && (((uintptr_t)p) & 15) == 0) {
      const uint4 q = *(const uint4*)p;
      const E* e = (const E*)&q;
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = to_f<E>(e[j]);
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = (r < rows && k + j < K) ? to_f<E>(p[j]) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) dst[(sg * VEC + j) * LD + r] = v[j];
  }
}
// dst[r][c] = src row r, columns h0..h0+HC-1 (natural layout), zero padded
template <typename E>
CMT_D void load_n(float* dst, const E* src, long long ld, int rows, int B, int b, int h0, int K) {
  constexpr int VEC = 16 / sizeof(E);
  constexpr int SEGS = HC / VEC;
  for (int i = threadIdx.x; i < P * SEGS; i += THREADS) {
    const int r = i / SEGS, sg = i % SEGS;
    const int k = h0 + sg * VEC;
    float v[VEC];
    const E* p = src + ((long long)r * B + b) * ld + k;
    if (r < rows && k + VEC <= K && (((uintptr_t)p) & 15) == 0) {
      const uint4 q = *(const uint4*)p;
      const E* e = (const E*)&q;
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = to_f<E>(e[j]);
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = (r < rows && k + j < K) ? to_f<E>(p[j]) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) dst[r * LD + sg * VEC + j] = v[j];
  }
}
// acc[i][j] += sum_{k<kn} A[k][i0+i] * Bm[k][j0+j]   (4x4 register tile)
CMT_D void mm44(float (&acc)[4][4], const float* A, const float* Bm, int i0, int j0, int kn) {
#pragma unroll 4
  for (int k = 0; k < kn; ++k) {
    const float4 a = *(const float4*)(A + k * LD + i0);
    const float4 c = *(const float4*)(Bm + k * LD + j0);
    const float av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], cv[j], acc[i][j]);
  }
}
CMT_D void zero44(float (&acc)[4][4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
}
// out[t][s] = sum_h X[t][h] Hs[s][h] over all h, into smem o[t*LD + s]
template <typename EX, typename EH>
CMT_D void scores(float* o, const EX* X, long long ldx, const EH* Hs, long long ldh, int T, int S, int B, int b, int H,
                  float* sX, float* sH) {
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float acc[4][4];
  zero44(acc);
  for (int k0 = 0; k0 < H; k0 += KC) {
    load_t(sX, X, ldx, T, B, b, k0, H);
    load_t(sH, Hs, ldh, S, B, b, k0, H);
    __syncthreads();
    mm44(acc, sX, sH, ty * 4, tx * 4, KC);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) o[(ty * 4 + i) * LD + tx * 4 + j] = acc[i][j];
}
inline size_t fwd_smem() { return sizeof(float) * (size_t)LD * (3 * P /*sc, aT, chunk*/); }
inline size_t bwd_smem() { return sizeof(float) * (size_t)LD * (4 * P /*da, al, ds, dsT*/ + 3 * P /*chunks*/); }
}  // namespace att

template <typename E>
__global__ void __launch_bounds__(att::THREADS) attn_fwd_tiled(const E* __restrict__ Hs, const E* __restrict__ U,
                                                               const float* __restrict__ src_mask, int S, int Tq, int B,
                                                               int H, float* __restrict__ alpha, E* __restrict__ ctx,
                                                               long long ldctx, int* __restrict__ status) {
  using namespace att;
  extern __shared__ float sm[];
  const int b = blockIdx.x;
  float* sc = sm;               // [t][s]
  float* aT = sc + P * LD;      // [s][t] alpha^T
  float* ch = aT + P * LD;      // [s][h] Hs chunk (also the score operands)
  float* sX = ch;               // [KC][t]
  float* sH = ch + KC * LD;     // [KC][s]
  scores(sc, U, H, Hs, H, Tq, S, B, b, H, sX, sH);
  __syncthreads();
  // masked softmax over s (layers.py:190-208): additive -1e9, max-subtract
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = warp; t < P; t += THREADS / 32) {
    float* row = sc + t * LD;
    if (t >= Tq) {
      for (int s = lane; s < P; s += 32) aT[s * LD + t] = 0.f;
      continue;
    }
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
    for (int s = lane; s < P; s += 32) {
      const float a = s < S ? row[s] / sum : 0.f;
      aT[s * LD + t] = a;
      if (s < S) alpha[((long long)b * Tq + t) * S + s] = a;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_SCORES);
  }
  __syncthreads();
  // ctx[t][h] = sum_s alpha[t][s] Hs[s][h]   (attention.py:67-75)
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  for (int h0 = 0; h0 < H; h0 += HC) {
    load_n(ch, Hs, H, S, B, b, h0, H);
    __syncthreads();
    float acc[4][4];
    zero44(acc);
    mm44(acc, aT, ch, ty * 4, tx * 4, S);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int t = ty * 4 + i;
      if (t >= Tq) continue;
      E* o = ctx + ((long long)t * B + b) * ldctx + h0 + tx * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (h0 + tx * 4 + j < H) o[j] = from_f<E>(acc[i][j]);
    }
    __syncthreads();
  }
}

// dC (fp32, row stride lddc) is dC_st[:, :H]; dHs (fp32) accumulates; dU = d(u) (E)
template <typename E>
__global__ void __launch_bounds__(att::THREADS) attn_bwd_tiled(const E* __restrict__ Hs, const E* __restrict__ U,
                                                               const float* __restrict__ alpha,
                                                               const float* __restrict__ dC, long long lddc, int S,
                                                               int Tq, int B, int H, float* __restrict__ dHs,
                                                               E* __restrict__ dU) {
  using namespace att;
  extern __shared__ float sm[];
  const int b = blockIdx.x;
  float* da = sm;             // [t][s]  d alpha, then d scores
  float* al = da + P * LD;    // [t][s]  alpha
  float* dsT = al + P * LD;   // [s][t]  d scores^T
  float* ds = dsT + P * LD;   // [t][s]  d scores
  float* cC = ds + P * LD;    // [t][h]  dC chunk  (also the score operands)
  float* cU = cC + P * LD;    // [t][h]  U chunk
  float* cH = cU + P * LD;    // [s][h]  Hs chunk
  // d alpha[t][s] = sum_h dC[t][h] Hs[s][h]   (attention.py:82-83)
  scores(da, dC, lddc, Hs, H, Tq, S, B, b, H, cC, cC + KC * LD);
  for (int i = threadIdx.x; i < P * P; i += THREADS) {
    const int t = i / P, s = i % P;
    al[t * LD + s] = (t < Tq && s < S) ? alpha[((long long)b * Tq + t) * S + s] : 0.f;
  }
  __syncthreads();
  // d scores = p (g - sum_s p g)   (layers.py:210-215); zero outside [Tq) x [S)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = warp; t < P; t += THREADS / 32) {
    const float* g = da + t * LD;
    const float* p = al + t * LD;
    float dot = 0.f;
    for (int s = lane; s < S; s += 32) dot += p[s] * g[s];
    dot = warp_sum(dot);
    for (int s = lane; s < P; s += 32) {
      const float v = (t < Tq && s < S) ? p[s] * (g[s] - dot) : 0.f;
      ds[t * LD + s] = v;
      dsT[s * LD + t] = v;
    }
  }
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  for (int h0 = 0; h0 < H; h0 += HC) {
    load_n(cC, dC, lddc, Tq, B, b, h0, H);
    load_n(cU, U, H, Tq, B, b, h0, H);
    load_n(cH, Hs, H, S, B, b, h0, H);
    __syncthreads();
    // dHs[s][h] += sum_t alpha[t][s] dC[t][h] + dscores[t][s] U[t][h]
    float acc[4][4];
    zero44(acc);
    mm44(acc, al, cC, ty * 4, tx * 4, Tq);
    mm44(acc, ds, cU, ty * 4, tx * 4, Tq);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int s = ty * 4 + i;
      if (s >= S) continue;
      float* o = dHs + ((long long)s * B + b) * H + h0 + tx * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (h0 + tx * 4 + j < H) o[j] += acc[i][j];
    }
    // du[t][h] = sum_s dscores[t][s] Hs[s][h]
    zero44(acc);
    mm44(acc, dsT, cH, ty * 4, tx * 4, S);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int t = ty * 4 + i;
      if (t >= Tq) continue;
      E* o = dU + ((long long)t * B + b) * H + h0 + tx * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (h0 + tx * 4 + j < H) o[j] = from_f<E>(acc[i][j]);
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// Split attention (one sentence spread over many CTAs; the score products'
// H reduction is split into HSPLIT slices whose partial sums are reduced in
// a fixed order, so results stay deterministic):
//   attn_scores_part   grid (B, H/HS): part[b][sp][t][s] = sum_{h in slice} X[t][h] Hs[s][h]
//   attn_softmax_fwd   grid B: scores = sum of slices, masked softmax -> alpha
//   attn_context       grid (B, H/HC): ctx[t][h] = sum_s alpha[t][s] Hs[s][h]
//   attn_dscores       grid B: dalpha = sum of slices; dscores = alpha (dalpha - sum alpha dalpha)
//   attn_bwd_chunk     grid (B, H/HC): dHs += alpha^T dC + dscores^T U, dU = dscores Hs
// Same arithmetic as attn_fwd_tiled / attn_bwd_tiled, spread over 16x the CTAs.
// ---------------------------------------------------------------------------
namespace att {
constexpr int HS = 128;  // h-slice of the score products per CTA
inline int nslices(int H) { return (H + HS - 1) / HS; }
}  // namespace att

template <typename EX, typename EH>
__global__ void __launch_bounds__(att::THREADS) attn_scores_part(const EX* __restrict__ X, long long ldx,
                                                                 const EH* __restrict__ Hs, int S, int Tq, int B, int H,
                                                                 float* __restrict__ part) {
  using namespace att;
  __shared__ __align__(16) float sX[KC * LD];
  __shared__ __align__(16) float sH[KC * LD];
  const int b = blockIdx.x, sp = blockIdx.y;
  const int h0 = sp * HS, h1 = min(H, h0 + HS);
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float acc[4][4];
  zero44(acc);
  for (int k0 = h0; k0 < h1; k0 += KC) {
    load_t(sX, X, ldx, Tq, B, b, k0, h1);
    load_t(sH, Hs, H, S, B, b, k0, h1);
    __syncthreads();
    mm44(acc, sX, sH, ty * 4, tx * 4, KC);
    __syncthreads();
  }
  float* o = part + ((size_t)b * gridDim.y + sp) * P * P;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *(float4*)(o + (ty * 4 + i) * P + tx * 4) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
}

__global__ void __launch_bounds__(att::THREADS) attn_softmax_fwd(const float* __restrict__ part, int nsp,
                                                                 const float* __restrict__ src_mask, int S, int Tq,
                                                                 int B, float* __restrict__ alpha,
                                                                 int* __restrict__ status) {
  using namespace att;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* pb = part + (size_t)b * nsp * P * P;
  for (int t = warp; t < Tq; t += THREADS / 32) {
    float v[2];
    float mx = -INFINITY;
    bool bad = false;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int s = lane + 32 * r;
      float a = 0.f;
      if (s < S) {
        for (int k = 0; k < nsp; ++k) a += pb[((size_t)k * P + t) * P + s];
        a += (1.f - src_mask[s * B + b]) * -1e9f;
        bad |= !isfinite(a);
        mx = fmaxf(mx, a);
      }
      v[r] = a;
    }
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int s = lane + 32 * r;
      v[r] = s < S ? expf(v[r] - mx) : 0.f;
      sum += v[r];
    }
    sum = warp_sum(sum);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int s = lane + 32 * r;
      if (s < S) alpha[((long long)b * Tq + t) * S + s] = v[r] / sum;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_SCORES);
  }
}

template <typename E>
__global__ void __launch_bounds__(att::THREADS) attn_context(const E* __restrict__ Hs, const float* __restrict__ alpha,
                                                             int S, int Tq, int B, int H, E* __restrict__ ctx,
                                                             long long ldctx) {
  using namespace att;
  __shared__ __align__(16) float aT[P * LD];  // [s][t]
  __shared__ __align__(16) float ch[P * LD];  // [s][h]
  const int b = blockIdx.x, h0 = blockIdx.y * HC;
  for (int i = threadIdx.x; i < P * P; i += THREADS) {
    const int s = i / P, t = i % P;
    aT[s * LD + t] = (s < S && t < Tq) ? alpha[((long long)b * Tq + t) * S + s] : 0.f;
  }
  load_n(ch, Hs, H, S, B, b, h0, H);
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float acc[4][4];
  zero44(acc);
  mm44(acc, aT, ch, ty * 4, tx * 4, S);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = ty * 4 + i;
    if (t >= Tq) continue;
    E* o = ctx + ((long long)t * B + b) * ldctx + h0 + tx * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (h0 + tx * 4 + j < H) o[j] = from_f<E>(acc[i][j]);
  }
}

__global__ void __launch_bounds__(att::THREADS) attn_dscores(const float* __restrict__ part, int nsp,
                                                             const float* __restrict__ alpha, int S, int Tq,
                                                             float* __restrict__ dsc) {
  using namespace att;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* pb = part + (size_t)b * nsp * P * P;
  for (int t = warp; t < Tq; t += THREADS / 32) {
    float g[2], p[2];
    float dot = 0.f;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int s = lane + 32 * r;
      float a = 0.f, pv = 0.f;
      if (s < S) {
        for (int k = 0; k < nsp; ++k) a += pb[((size_t)k * P + t) * P + s];
        pv = alpha[((long long)b * Tq + t) * S + s];
      }
      g[r] = a;
      p[r] = pv;
      dot += pv * a;
    }
    dot = warp_sum(dot);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int s = lane + 32 * r;
      if (s < S) dsc[((long long)b * Tq + t) * S + s] = p[r] * (g[r] - dot);
    }
  }
}

template <typename E>
__global__ void __launch_bounds__(att::THREADS) attn_bwd_chunk(const E* __restrict__ Hs, const E* __restrict__ U,
                                                               const float* __restrict__ alpha,
                                                               const float* __restrict__ dsc,
                                                               const float* __restrict__ dC, long long lddc, int S,
                                                               int Tq, int B, int H, float* __restrict__ dHs,
                                                               E* __restrict__ dU) {
  using namespace att;
  extern __shared__ float sm[];
  float* al = sm;             // [t][s]
  float* ds = al + P * LD;    // [t][s]
  float* dsT = ds + P * LD;   // [s][t]
  float* cC = dsT + P * LD;   // [t][h]
  float* cU = cC + P * LD;    // [t][h]
  float* cH = cU + P * LD;    // [s][h]
  const int b = blockIdx.x, h0 = blockIdx.y * HC;
  for (int i = threadIdx.x; i < P * P; i += THREADS) {
    const int t = i / P, s = i % P;
    const bool ok = t < Tq && s < S;
    const long long o = ((long long)b * Tq + t) * S + s;
    al[t * LD + s] = ok ? alpha[o] : 0.f;
    const float d = ok ? dsc[o] : 0.f;
    ds[t * LD + s] = d;
    dsT[s * LD + t] = d;
  }
  load_n(cC, dC, lddc, Tq, B, b, h0, H);
  load_n(cU, U, H, Tq, B, b, h0, H);
  load_n(cH, Hs, H, S, B, b, h0, H);
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float acc[4][4];
  zero44(acc);
  mm44(acc, al, cC, ty * 4, tx * 4, Tq);
  mm44(acc, ds, cU, ty * 4, tx * 4, Tq);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int s = ty * 4 + i;
    if (s >= S) continue;
    float* o = dHs + ((long long)s * B + b) * H + h0 + tx * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (h0 + tx * 4 + j < H) o[j] += acc[i][j];
  }
  zero44(acc);
  mm44(acc, dsT, cH, ty * 4, tx * 4, S);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = ty * 4 + i;
    if (t >= Tq) continue;
    E* o = dU + ((long long)t * B + b) * H + h0 + tx * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (h0 + tx * 4 + j < H) o[j] = from_f<E>(acc[i][j]);
  }
}


// ---------------------------------------------------------------------------
// Tiled split attention for S, T <= 128 (used for every length <= 128): the
// (t, s) plane is cut into 64 x 64 tiles and every product gets its own grid
// axis over tiles, so longer sentences (c5: S = T = 80) stay on the same
// register-tiled path.  The dHs and dU products are separate kernels.
// ---------------------------------------------------------------------------
namespace att2 {
using att::HC;
using att::KC;
using att::LD;
using att::THREADS;
constexpr int P = 64;       // tile edge
constexpr int MAXL = 128;   // longest S / T handled
CMT_HD int tiles(int n) { return (n + P - 1) / P; }

// dst[k][r] = src row r0 + r (r < 64), columns k0..k0+KC-1, zero padded
template <typename E>
CMT_D void load_t_tile(float* dst, const E* src, long long ld, int r0, int rows, int B, int b, int k0, int K) {
  constexpr int VEC = 16 / sizeof(E);
  constexpr int SEGS = KC / VEC;
  for (int i = threadIdx.x; i < P * SEGS; i += THREADS) {
    const int r = i / SEGS, sg = i % SEGS;
    const int k = k0 + sg * VEC;
    const int gr = r0 + r;
    float v[VEC];
    const E* p = src + ((long long)gr * B + b) * ld + k;
    if (gr < rows && k + VEC <= K && (((uintptr_t)p) & 15) == 0) {
      const uint4 q = *(const uint4*)p;
      const E* e = (const E*)&q;
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = to_f<E>(e[j]);
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = (gr < rows && k + j < K) ? to_f<E>(p[j]) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) dst[(sg * VEC + j) * LD + r] = v[j];
  }
}
// dst[r][c] = src row r (r < npad), columns h0..h0+HC-1, zero padded
template <typename E>
CMT_D void load_n_rows(float* dst, const E* src, long long ld, int npad, int rows, int B, int b, int h0, int K) {
  constexpr int VEC = 16 / sizeof(E);
  constexpr int SEGS = HC / VEC;
  for (int i = threadIdx.x; i < npad * SEGS; i += THREADS) {
    const int r = i / SEGS, sg = i % SEGS;
    const int k = h0 + sg * VEC;
    float v[VEC];
    const E* p = src + ((long long)r * B + b) * ld + k;
    if (r < rows && k + VEC <= K && (((uintptr_t)p) & 15) == 0) {
      const uint4 q = *(const uint4*)p;
      const E* e = (const E*)&q;
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = to_f<E>(e[j]);
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = (r < rows && k + j < K) ? to_f<E>(p[j]) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) dst[r * LD + sg * VEC + j] = v[j];
  }
}
}  // namespace att2

// part[b][sp][t][s] (t < Tp, s < Sp padded to 64) = sum_{h in slice sp} X[t][h] Hs[s][h]
template <typename EX, typename EH>
__global__ void __launch_bounds__(att::THREADS) attn2_scores_part(const EX* __restrict__ X, long long ldx,
                                                                  const EH* __restrict__ Hs, int S, int Tq, int B,
                                                                  int H, float* __restrict__ part) {
  using namespace att2;
  __shared__ __align__(16) float sX[KC * LD];
  __shared__ __align__(16) float sH[KC * LD];
  const int b = blockIdx.x, sp = blockIdx.y, nsp = gridDim.y;
  const int ts = tiles(S), Tp = tiles(Tq) * P, Sp = ts * P;
  const int t0 = (blockIdx.z / ts) * P, s0 = (blockIdx.z % ts) * P;
  const int h0 = sp * att::HS, h1 = min(H, h0 + att::HS);
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float acc[4][4];
  att::zero44(acc);
  for (int k0 = h0; k0 < h1; k0 += KC) {
    load_t_tile(sX, X, ldx, t0, Tq, B, b, k0, h1);
    load_t_tile(sH, Hs, H, s0, S, B, b, k0, h1);
    __syncthreads();
    att::mm44(acc, sX, sH, ty * 4, tx * 4, KC);
    __syncthreads();
  }
  float* o = part + ((size_t)b * nsp + sp) * Tp * Sp;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *(float4*)(o + (size_t)(t0 + ty * 4 + i) * Sp + s0 + tx * 4) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
}

// mode 0: alpha = masked softmax of the summed scores; mode 1: dscores = alpha (g - sum alpha g)
__global__ void __launch_bounds__(att::THREADS) attn2_rows(const float* __restrict__ part, int nsp,
                                                           const float* __restrict__ src_mask, int S, int Tq, int B,
                                                           float* __restrict__ alpha, float* __restrict__ dsc,
                                                           int mode, int* __restrict__ status) {
  using namespace att2;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Tp = tiles(Tq) * P, Sp = tiles(S) * P;
  const float* pb = part + (size_t)b * nsp * Tp * Sp;
  for (int t = warp; t < Tq; t += THREADS / 32) {
    float v[MAXL / 32], pv[MAXL / 32];
#pragma unroll
    for (int r = 0; r < MAXL / 32; ++r) {
      const int s = lane + 32 * r;
      float a = 0.f;
      if (s < S)
        for (int k = 0; k < nsp; ++k) a += pb[((size_t)k * Tp + t) * Sp + s];
      v[r] = a;
      pv[r] = (mode == 1 && s < S) ? alpha[((long long)b * Tq + t) * S + s] : 0.f;
    }
    if (mode == 0) {
      float mx = -INFINITY;
      bool bad = false;
#pragma unroll
      for (int r = 0; r < MAXL / 32; ++r) {
        const int s = lane + 32 * r;
        if (s < S) {
          v[r] += (1.f - src_mask[s * B + b]) * -1e9f;
          bad |= !isfinite(v[r]);
          mx = fmaxf(mx, v[r]);
        }
      }
      mx = warp_max(mx);
      float sum = 0.f;
#pragma unroll
      for (int r = 0; r < MAXL / 32; ++r) {
        const int s = lane + 32 * r;
        v[r] = s < S ? expf(v[r] - mx) : 0.f;
        sum += v[r];
      }
      sum = warp_sum(sum);
#pragma unroll
      for (int r = 0; r < MAXL / 32; ++r) {
        const int s = lane + 32 * r;
        if (s < S) alpha[((long long)b * Tq + t) * S + s] = v[r] / sum;
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_SCORES);
    } else {
      float dot = 0.f;
#pragma unroll
      for (int r = 0; r < MAXL / 32; ++r) dot += pv[r] * v[r];
      dot = warp_sum(dot);
#pragma unroll
      for (int r = 0; r < MAXL / 32; ++r) {
        const int s = lane + 32 * r;
        if (s < S) dsc[((long long)b * Tq + t) * S + s] = pv[r] * (v[r] - dot);
      }
    }
  }
}

// out[t][h] (t-tile blockIdx.z) = sum_s W[t][s] Hs[s][h]; W = alpha (ctx) or dscores (dU)
template <typename E>
__global__ void __launch_bounds__(att::THREADS) attn2_ws_hs(const E* __restrict__ Hs, const float* __restrict__ W,
                                                            int S, int Tq, int B, int H, E* __restrict__ out,
                                                            long long ldo) {
  using namespace att2;
  extern __shared__ float sm[];
  const int Sp = tiles(S) * P;
  float* wT = sm;            // [s][t-local]
  float* ch = sm + Sp * LD;  // [s][h]
  const int b = blockIdx.x, h0 = blockIdx.y * HC, t0 = blockIdx.z * P;
  for (int i = threadIdx.x; i < Sp * P; i += THREADS) {
    const int s = i / P, t = i % P;
    wT[s * LD + t] = (s < S && t0 + t < Tq) ? W[((long long)b * Tq + t0 + t) * S + s] : 0.f;
  }
  load_n_rows(ch, Hs, H, Sp, S, B, b, h0, H);
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float acc[4][4];
  att::zero44(acc);
  att::mm44(acc, wT, ch, ty * 4, tx * 4, S);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + ty * 4 + i;
    if (t >= Tq) continue;
    E* o = out + ((long long)t * B + b) * ldo + h0 + tx * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (h0 + tx * 4 + j < H) o[j] = from_f<E>(acc[i][j]);
  }
}

// dHs[s][h] (s-tile blockIdx.z) += sum_t alpha[t][s] dC[t][h] + dscores[t][s] U[t][h]
template <typename E>
__global__ void __launch_bounds__(att::THREADS) attn2_dhs(const E* __restrict__ U, const float* __restrict__ alpha,
                                                          const float* __restrict__ dsc, const float* __restrict__ dC,
                                                          long long lddc, int S, int Tq, int B, int H,
                                                          float* __restrict__ dHs) {
  using namespace att2;
  extern __shared__ float sm[];
  const int Tp = tiles(Tq) * P;
  float* al = sm;             // [t][s-local]
  float* ds = al + Tp * LD;   // [t][s-local]
  float* cC = ds + Tp * LD;   // [t][h]
  float* cU = cC + Tp * LD;   // [t][h]
  const int b = blockIdx.x, h0 = blockIdx.y * HC, s0 = blockIdx.z * P;
  for (int i = threadIdx.x; i < Tp * P; i += THREADS) {
    const int t = i / P, s = i % P;
    const bool ok = t < Tq && s0 + s < S;
    const long long o = ((long long)b * Tq + t) * S + s0 + s;
    al[t * LD + s] = ok ? alpha[o] : 0.f;
    ds[t * LD + s] = ok ? dsc[o] : 0.f;
  }
  load_n_rows(cC, dC, lddc, Tp, Tq, B, b, h0, H);
  load_n_rows(cU, U, H, Tp, Tq, B, b, h0, H);
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  float acc[4][4];
  att::zero44(acc);
  att::mm44(acc, al, cC, ty * 4, tx * 4, Tq);
  att::mm44(acc, ds, cU, ty * 4, tx * 4, Tq);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int s = s0 + ty * 4 + i;
    if (s >= S) continue;
    float* o = dHs + ((long long)s * B + b) * H + h0 + tx * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (h0 + tx * 4 + j < H) o[j] += acc[i][j];
  }
}

}  // namespace cmt
