// GEMM family for the train step.
//
// Logical contract: C[m][n] = epilogue( sum_k A(m,k) * B(n,k) ).
//   A(m,k) lives at A + m*lda + k (K-major) or A + k*lda + m (MN-major),
//   B(n,k) likewise.  Every GEMM of the step maps onto
//   one of (A K-major, B MN-major) [forward: X @ W], (K, K) [dgrad: dY @ W^T]
//   or (MN, MN) [wgrad: X^T @ dY] with weights kept in the reference's natural
//   (dim_in, dim_out) layout — no transposed weight copies.
//
// Production (bf16): persistent warp-specialised tcgen05 kernel.  TMA loads
// 128B-swizzled tiles into a multi-stage smem ring, one elected thread issues
// tcgen05.mma (M=128, N=BN, K=16) into a double-buffered TMEM accumulator,
// four epilogue warps drain TMEM with tcgen05.ld and run a fused epilogue
// functor (bias/tanh/dropout-mask/accumulate, or the LSTM cell forward /
// backward) while the next tile's MMAs proceed.
//
// Validation (fp32): a tiled SIMT kernel with the *same* epilogue functors, so
// the fp32 validation mode exercises identical orchestration and cell math.
#pragma once
#include "ptx.cuh"

namespace cmt {

// ---------------------------------------------------------------------------
// Epilogues.  apply(m, n0, v, M, N): v holds the 32 accumulator values of row
// m, columns n0..n0+31 (columns >= N must be ignored).
// ---------------------------------------------------------------------------

struct EpiStore {
  void* C = nullptr;
  long long ldc = 0;
  int c_bf16 = 0;
  int beta = 0;                  // C += result (fp32 C only)
  const float* add = nullptr;    // result += add[m*ld_add + n]
  long long ld_add = 0;
  const float* bias = nullptr;   // per column
  int act = 0;                   // 1: tanh
  const uint8_t* dmask = nullptr;  // dropout keep-mask (applied after act)
  long long ld_dmask = 0;
  float dscale = 1.f;
  const float* tgrad_y = nullptr;  // multiply by (1 - y^2): tanh' from its output
  long long ld_tgrad = 0;

  // x[j] = epilogue value of (m, n0 + j); rows m >= M read no row operands.
  // F (compile-time): 1 bias, 2 tanh, 4 dropout mask, 8 tanh' from output, 16 add;
  // F = 63: any combination, each stage gated at run time.
  // Every global load of the chunk is issued up front (vectorised where the
  // row is 16-byte aligned) and the element loop is branch-free.
  // the chunk's 32 bias values; issued by the epilogue before its TMEM load so
  // the two latencies overlap (compute_t then takes them from `pb`)
  CMT_D void load_bias(int n0, int N, float* bv) const {
    if (n0 + 32 <= N && (((uintptr_t)(bias + n0)) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) *(float4*)&bv[4 * q] = __ldg((const float4*)(bias + n0) + q);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) bv[j] = (n0 + j < N) ? __ldg(bias + n0 + j) : 0.f;
    }
  }
  template <int F>
  CMT_D void compute_t(int m, int n0, const float* v, int M, int N, float* x, const float* pb = nullptr) const {
    const bool full = (n0 + 32 <= N);
    const bool row_ok = m < M;
    const long long rm = row_ok ? (long long)m : 0;
    const int fl = (F & 32) ? flags() : F;
    float bv[(F & 1) ? 32 : 1], tg[(F & 8) ? 32 : 1], ad[(F & 16) ? 32 : 1];
    uint8_t km[(F & 4) ? 32 : 1];
    if ((F & 1) && (fl & 1) && pb) {
#pragma unroll
      for (int j = 0; j < 32; ++j) bv[j] = pb[j];
    } else if ((F & 1) && (fl & 1)) {
      if (full && (((uintptr_t)(bias + n0)) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) *(float4*)&bv[4 * q] = __ldg((const float4*)(bias + n0) + q);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) bv[j] = (n0 + j < N) ? __ldg(bias + n0 + j) : 0.f;
      }
    }
    if ((F & 4) && (fl & 4)) {
      const uint8_t* dm = dmask + rm * ld_dmask + n0;
      if (row_ok && full && (((uintptr_t)dm) & 15) == 0) {
        *(uint4*)&km[0] = *(const uint4*)dm;
        *(uint4*)&km[16] = *(const uint4*)(dm + 16);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) km[j] = (row_ok && n0 + j < N) ? dm[j] : 0;
      }
    }
    if ((F & 8) && (fl & 8)) {
      const float* ty = tgrad_y + rm * ld_tgrad + n0;
      if (row_ok && full && (((uintptr_t)ty) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) *(float4*)&tg[4 * q] = *((const float4*)ty + q);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) tg[j] = (row_ok && n0 + j < N) ? ty[j] : 0.f;
      }
    }
    if ((F & 16) && (fl & 16)) {
      const float* aa = add + rm * ld_add + n0;
      if (row_ok && full && (((uintptr_t)aa) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) *(float4*)&ad[4 * q] = *((const float4*)aa + q);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) ad[j] = (row_ok && n0 + j < N) ? aa[j] : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float t = v[j];
      if ((F & 1) && (fl & 1)) t += bv[(F & 1) ? j : 0];
      if ((F & 2) && (fl & 2)) t = c_bf16 ? ptx::tanh_fast(t) : tanhf(t);
      if ((F & 4) && (fl & 4)) t = km[(F & 4) ? j : 0] ? t * dscale : 0.f * t;
      if ((F & 8) && (fl & 8)) t *= (1.f - tg[(F & 8) ? j : 0] * tg[(F & 8) ? j : 0]);
      if ((F & 16) && (fl & 16)) t += ad[(F & 16) ? j : 0];
      x[j] = t;
    }
  }
  CMT_D int flags() const {
    return (bias ? 1 : 0) | (act == 1 ? 2 : 0) | (dmask ? 4 : 0) | (tgrad_y ? 8 : 0) | (add ? 16 : 0);
  }
  CMT_D void compute(int m, int n0, const float* v, int M, int N, float* x, const float* pb = nullptr) const {
    switch (flags()) {
      case 0: compute_t<0>(m, n0, v, M, N, x); break;
      case 1: compute_t<1>(m, n0, v, M, N, x, pb); break;
      case 2: compute_t<2>(m, n0, v, M, N, x); break;
      case 3: compute_t<3>(m, n0, v, M, N, x, pb); break;
      case 4: compute_t<4>(m, n0, v, M, N, x); break;
      case 8: compute_t<8>(m, n0, v, M, N, x); break;
      case 12: compute_t<12>(m, n0, v, M, N, x); break;
      case 16: compute_t<16>(m, n0, v, M, N, x); break;
      default: compute_any(m, n0, v, M, N, x, pb);
    }
  }
  // any other stage combination: the same stages, each operand loaded per
  // element (no 32-wide staging arrays, so this rarely-used path adds no
  // register pressure to the kernel)
  CMT_D void compute_any(int m, int n0, const float* v, int M, int N, float* x, const float* pb) const {
    const bool row_ok = m < M;
    const long long rm = row_ok ? (long long)m : 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const bool ok = row_ok && n0 + j < N;
      float t = v[j];
      if (bias) t += pb ? pb[j] : (n0 + j < N ? __ldg(bias + n0 + j) : 0.f);
      if (act == 1) t = c_bf16 ? ptx::tanh_fast(t) : tanhf(t);
      if (dmask) t = (ok && dmask[rm * ld_dmask + n0 + j]) ? t * dscale : 0.f * t;
      if (tgrad_y) {
        const float ty = ok ? tgrad_y[rm * ld_tgrad + n0 + j] : 0.f;
        t *= (1.f - ty * ty);
      }
      if (add) t += ok ? add[rm * ld_add + n0 + j] : 0.f;
      x[j] = t;
    }
  }

  CMT_D void apply(int m, int n0, const float* v, int M, int N) const {
    const bool full = (n0 + 32 <= N);
    float x[32];
    compute(m, n0, v, M, N, x);
    long long base = (long long)m * ldc + n0;
    if (c_bf16) {
      bf16* c = (bf16*)C + base;
      if (full && ((((uintptr_t)c) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          __align__(16) bf16 tmp[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) tmp[j] = __float2bfloat16_rn(x[q * 8 + j]);
          *(uint4*)(c + q * 8) = *(uint4*)tmp;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (n0 + j < N) c[j] = __float2bfloat16_rn(x[j]);
      }
    } else {
      float* c = (float*)C + base;
      if (full && ((((uintptr_t)c) & 15) == 0)) {
        if (beta) {
          float4 old[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) old[q] = *(float4*)(c + q * 4);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            x[q * 4] += old[q].x; x[q * 4 + 1] += old[q].y; x[q * 4 + 2] += old[q].z; x[q * 4 + 3] += old[q].w;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) *(float4*)(c + q * 4) = make_float4(x[q * 4], x[q * 4 + 1], x[q * 4 + 2], x[q * 4 + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (n0 + j < N) c[j] = beta ? c[j] + x[j] : x[j];
      }
    }
  }
};

// LSTM forward cell fused into the recurrent GEMM of step t
// (reference layers.py:344-363 cell, layers.py:453-464 mask gating).
// Gate columns are interleaved: column 4*j+q is gate q (i,f,g,o) of unit j.
struct EpiLstmFwd {
  const float* ux;      // [rows][4H]  hoisted W_x x_t + b (row = row0 + m)
  const void* hprev;    // act [rows][H] (h_{t-1}, row = row0 + m)
  const float* cprev;   // [rows][H]
  void* y;              // act [rows][H]  h_t (masked carry)
  float* cst;           // [rows][H]      c_t (masked carry)
  float* acts;          // [rows][4H]     i,f,g,o
  float* tcache;        // [rows][H]      tanh(c_new)
  const float* mask;    // [B] for this step, or null (decoder: unmasked)
  long long row0;
  int H;
  int act_bf16;

  CMT_D void apply(int m, int n0, const float* v, int M, int N) const {
    long long row = row0 + m;
    const float* uxr = ux + row * 4LL * H;
    float mk = mask ? mask[m] : 1.f;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      int gc = n0 + 4 * jj;
      if (gc >= N) break;
      int j = gc >> 2;
      float4 u4 = *(const float4*)(uxr + gc);
      float gi = sigmoidf_(v[4 * jj + 0] + u4.x);
      float gf = sigmoidf_(v[4 * jj + 1] + u4.y);
      float gg = tanhf(v[4 * jj + 2] + u4.z);
      float go = sigmoidf_(v[4 * jj + 3] + u4.w);
      float cp = cprev[row * H + j];
      float hp = act_bf16 ? __bfloat162float(((const bf16*)hprev)[row * H + j]) : ((const float*)hprev)[row * H + j];
      float cn = __fadd_rn(__fmul_rn(gf, cp), __fmul_rn(gi, gg));
      float tcn = tanhf(cn);
      float hn = __fmul_rn(go, tcn);
      float h = hn, c = cn;
      if (mask) {
        h = mk * hn + (1.f - mk) * hp;
        c = mk * cn + (1.f - mk) * cp;
      }
      *(float4*)(acts + row * 4LL * H + gc) = make_float4(gi, gf, gg, go);
      tcache[row * H + j] = tcn;
      cst[row * H + j] = c;
      if (act_bf16) ((bf16*)y)[row * H + j] = __float2bfloat16_rn(h);
      else ((float*)y)[row * H + j] = h;
    }
  }
};

// LSTM cell backward at time t fused into the dh GEMM (acc = W_h dU_{t_next}).
// reference layers.py:366-395 (cell) and layers.py:477-490 (mask split).
struct EpiLstmBwd {
  const float* dy;      // [rows][H] grad of this layer's output (row = row0 + m)
  float* dhc;           // [B][H] carry (1-m) dh from the later step, in/out
  float* dc;            // [B][H] cell grad carry, in/out
  const float* acts;    // [rows][4H]
  const float* tcache;  // [rows][H]
  const float* cprev;   // [rows][H]
  const float* mask;    // [B] or null
  void* dU;             // act [rows][4H]
  long long row0;
  int H;
  int act_bf16;

  CMT_D void apply(int m, int n0, const float* v, int M, int N) const {
    long long row = row0 + m;
    float mk = mask ? mask[m] : 1.f;
    for (int jj = 0; jj < 32; ++jj) {
      int j = n0 + jj;
      if (j >= N) break;
      long long bi = (long long)m * H + j;
      float dh = v[jj] + dhc[bi] + dy[row * H + j];
      float dcin = dc[bi];
      float dhn = dh, dcn = dcin, dhcar = 0.f, dccar = 0.f;
      if (mask) {
        dhn = mk * dh; dcn = mk * dcin;
        dhcar = (1.f - mk) * dh; dccar = (1.f - mk) * dcin;
      }
      float4 a = *(const float4*)(acts + row * 4LL * H + 4 * j);  // i f g o
      float tc = tcache[row * H + j];
      float cp = cprev[row * H + j];
      float dct = dhn * a.w * (1.f - tc * tc) + dcn;
      float di = dct * a.z * (a.x * (1.f - a.x));
      float df = dct * cp * (a.y * (1.f - a.y));
      float dg = dct * a.x * (1.f - a.z * a.z);
      float dO = dhn * tc * (a.w * (1.f - a.w));
      long long o = row * 4LL * H + 4 * j;
      if (act_bf16) {
        __align__(8) bf16 t4[4] = {__float2bfloat16_rn(di), __float2bfloat16_rn(df), __float2bfloat16_rn(dg),
                                   __float2bfloat16_rn(dO)};
        *(uint2*)((bf16*)dU + o) = *(uint2*)t4;
      } else {
        *(float4*)((float*)dU + o) = make_float4(di, df, dg, dO);
      }
      dc[bi] = dct * a.y + dccar;
      dhc[bi] = dhcar;
    }
  }
};

// After the last BPTT step: grads of the initial state (layers.py:491-493).
struct EpiInitGrad {
  float* dh0;           // [B][H]
  float* dc0;           // [B][H]
  const float* dhc;
  const float* dc;
  int H;
  CMT_D void apply(int m, int n0, const float* v, int M, int N) const {
    for (int jj = 0; jj < 32; ++jj) {
      int j = n0 + jj;
      if (j >= N) break;
      long long bi = (long long)m * H + j;
      dh0[bi] = v[jj] + dhc[bi];
      dc0[bi] = dc[bi];
    }
  }
};

// ---------------------------------------------------------------------------
// tcgen05 persistent GEMM (bf16 -> fp32)
//
// CG = 1: one CTA per 128 x BN tile.
// CG = 2: a CTA pair (cluster of 2, cta_group::2) per 256 x BN tile.  Each CTA
//   TMA-loads its own 128 rows of A and BN/2 columns of B; the leader's single
//   MMA thread issues M=256 tcgen05.mma that read both CTAs' smem, so each SM
//   streams half the B bytes of the CG=1 kernel for the same MMA rate (the
//   1-CTA 128x256 tile needs ~96 B/clk/SM of TMA, the pair 64 B/clk/SM).
//   Stage completion bytes of both CTAs land on the leader's full barrier;
//   MMA commits multicast the stage-empty / accumulator-full signals to both
//   CTAs; both CTAs' epilogue warps release the accumulator on the leader.
// ---------------------------------------------------------------------------
namespace tc {
constexpr int BM = 128;
constexpr int BK = 64;
constexpr int NUM_THREADS = 384;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-11 epilogue (2 per SMSP)
constexpr int EPI_WARPS = 8;

constexpr int STG_BYTES = 32 * 32 * 4;  // one epilogue staging buffer: 32 rows x 128 B
template <int BN, int CG = 1, int ST = 0>
struct Cfg {
  static constexpr int BNC = BN / CG;  // B columns held by one CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BNC * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGING = ST ? EPI_WARPS * 2 * STG_BYTES : 0;  // double-buffered per epilogue warp
  static constexpr int STAGES_RAW = (ST ? (227 * 1024 - 2048 - STAGING) : 200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = (2 * BN) <= 32 ? 32 : (2 * BN) <= 64 ? 64 : (2 * BN) <= 128 ? 128 : (2 * BN) <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 /*align slack*/ + STAGES * STAGE_BYTES + STAGING + 1024 /*barriers*/;
  static constexpr int TILE_M = BM * CG;
};
}  // namespace tc

// Work distribution of the persistent GEMM.  ks >= 1: unit u takes work items
// u, u+nunits, ... where item w = (tile w / ks, K slice w % ks).  ks == -1
// (owner/helper stream-K, for tiles < units): unit t < tiles owns k-blocks
// [0, a) of tile t; the nunits - tiles helper units each take the tails
// [a, num_kb) of tph consecutive tiles, with a chosen so owners and helpers
// carry equal k-block loads.  Every tile then has exactly two pieces, both
// TMA-reduce-added into a zeroed C (order-independent: fp32 + commutes).
// Each role (TMA, MMA, epilogue) walks the same sequence.
struct GemmWork {
  int tile, kb0, nk;
  int w, step, end, ks, num_kb, a;
  bool helper;
  CMT_D GemmWork(int unit, int nunits, int num_tiles, int ks_, int num_kb_) {
    ks = ks_;
    num_kb = num_kb_;
    helper = false;
    if (ks_ < 0) {
      const int nh = nunits - num_tiles;  // > 0 (host guarantees tiles < units)
      const int tph = (num_tiles + nh - 1) / nh;
      a = num_kb_ * tph / (tph + 1);
      if (unit < num_tiles) {
        w = unit; end = unit + 1; step = 1;
      } else {
        helper = true;
        w = (unit - num_tiles) * tph;
        end = min(num_tiles, w + tph);
        step = 1;
      }
    } else {
      w = unit;
      step = nunits;
      end = num_tiles * ks_;
      a = 0;
    }
  }
  CMT_D bool next() {
    if (w >= end) return false;
    if (ks < 0) {
      tile = w;
      kb0 = helper ? a : 0;
      nk = helper ? num_kb - a : a;
    } else {
      tile = w / ks;
      const int sp = w % ks;
      kb0 = sp * num_kb / ks;
      nk = (sp + 1) * num_kb / ks - kb0;
    }
    w += step;
    return true;
  }
};

// ST = 1 (EpiStore only): the epilogue stages each warp's 32x32 result block
// in 128B/64B-swizzled smem and writes it with a TMA store (or a TMA
// reduce-add for beta) instead of per-row global stores.
template <int BN, int A_MN, int B_MN, class Epi, int CG = 1, int ST = 0>
__global__ void __launch_bounds__(tc::NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, int M, int N, int K, Epi epi, int opt, int ks) {
  using C = tc::Cfg<BN, CG, ST>;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * C::A_BYTES;
  uint8_t* stg = smem + S * C::STAGE_BYTES;  // epilogue staging (ST), 1024-aligned
  uint64_t* full = (uint64_t*)(stg + C::STAGING);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? ptx::cluster_rank() : 0u;
  const int unit = (CG == 2) ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // tile-processing unit (CTA or pair)
  const int nunits = (CG == 2) ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int tiles_m = (M + C::TILE_M - 1) / C::TILE_M;
  const int tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = (K + tc::BK - 1) / tc::BK;
  // split-K (ST only, linear epilogues): work unit w -> tile w / ks, K slice w % ks;
  // every slice reduce-adds its partial tile into C

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if (ST) ptx::prefetch_tmap(&tmC);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], tc::EPI_WARPS * CG);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2) ptx::tmem_alloc_cg2(tmem_slot, C::TMEM_COLS);
    else ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync_all();
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && num_kb > 0) {
      // ===== TMA producer (both CTAs of a pair load their own halves) =====
      int stage = 0;
      uint32_t phase = 0;
      GemmWork wk(unit, nunits, num_tiles, ks, num_kb);
      while (wk.next()) {
        const int tile = wk.tile;
        const int tm_ = (opt & 2) ? tile / tiles_n : tile % tiles_m;
        const int tn_ = (opt & 2) ? tile % tiles_n : tile / tiles_m;
        const int m0 = tm_ * C::TILE_M + (int)rank * tc::BM;
        const int n0 = tn_ * BN + (int)rank * C::BNC;
        const int kbl = wk.kb0, nk = wk.nk;
        for (int kk_ = 0; kk_ < nk; ++kk_) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * C::A_BYTES;
          uint8_t* b = sB + stage * C::B_BYTES;
          // stagger the K order per tile so concurrent CTAs sharing an operand
          // tile do not request the same L2 lines at the same moment
          const int k0 = (kbl + ((opt & 1) ? kk_ : (kk_ + tile) % nk)) * tc::BK;
          if constexpr (CG == 2) {
            const uint32_t fb = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
            if (rank == 0) ptx::mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            if (A_MN) {
              ptx::tma_load_2d_cg2(&tmA, fb, a, m0, k0);
              ptx::tma_load_2d_cg2(&tmA, fb, a + 64 * tc::BK * 2, m0 + 64, k0);
            } else {
              ptx::tma_load_2d_cg2(&tmA, fb, a, k0, m0);
            }
            if (B_MN) {
#pragma unroll
              for (int q = 0; q < C::BNC / 64; ++q)
                ptx::tma_load_2d_cg2(&tmB, fb, b + q * 64 * tc::BK * 2, n0 + q * 64, k0);
            } else {
              ptx::tma_load_2d_cg2(&tmB, fb, b, k0, n0);
            }
          } else {
            if (A_MN) {
              ptx::tma_load_2d(&tmA, &full[stage], a, m0, k0);
              ptx::tma_load_2d(&tmA, &full[stage], a + 64 * tc::BK * 2, m0 + 64, k0);
            } else {
              ptx::tma_load_2d(&tmA, &full[stage], a, k0, m0);
            }
            if (B_MN) {
#pragma unroll
              for (int q = 0; q < BN / 64; ++q)
                ptx::tma_load_2d(&tmB, &full[stage], b + q * 64 * tc::BK * 2, n0 + q * 64, k0);
            } else {
              ptx::tma_load_2d(&tmB, &full[stage], b, k0, n0);
            }
            ptx::mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && num_kb > 0 && rank == 0) {
      // ===== MMA issuer (the leader CTA of a pair) =====
      const uint32_t idesc = ptx::idesc_bf16(C::TILE_M, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      GemmWork wk(unit, nunits, num_tiles, ks, num_kb);
      for (; wk.next(); ++iter) {
        const int nk = wk.nk;
        const int buf = iter & 1;
        const uint32_t aphase = (iter >> 1) & 1;
        ptx::mbar_wait(&tempty[buf], aphase ^ 1);
        ptx::tc_fence_after();
        const uint32_t dtm = tmem_base + buf * BN;
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = ptx::smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < tc::BK / 16; ++kk) {
            uint64_t ad = A_MN ? ptx::smem_desc_sw128(a_addr + kk * 2048, 64 * tc::BK * 2, 1024)
                               : ptx::smem_desc_sw128(a_addr + kk * 32, 16, 1024);
            uint64_t bd = B_MN ? ptx::smem_desc_sw128(b_addr + kk * 2048, 64 * tc::BK * 2, 1024)
                               : ptx::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
            if constexpr (CG == 2) ptx::umma_bf16_cg2(dtm, ad, bd, idesc, (kb | kk) ? 1u : 0u);
            else ptx::umma_bf16(dtm, ad, bd, idesc, (kb | kk) ? 1u : 0u);
          }
          if constexpr (CG == 2) {
            ptx::umma_commit_cg2_mc(&empty[stage], 3);
            if (kb == nk - 1) ptx::umma_commit_cg2_mc(&tfull[buf], 3);
          } else {
            ptx::umma_commit(&empty[stage]);
            if (kb == nk - 1) ptx::umma_commit(&tfull[buf]);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: warps 4-7 drain the first half of the columns, 8-11 the second =====
    const int q = warp & 3;  // TMEM lane quarter accessible by this warp
    constexpr int NCH = BN / 32;
    const int c_lo = (warp < 8) ? 0 : (NCH + 1) / 2;
    const int c_hi = (warp < 8) ? (NCH + 1) / 2 : NCH;
    const uint32_t tempty_leader0 = (CG == 2) ? ptx::mapa(ptx::smem_u32(&tempty[0]), 0) : 0u;
    uint8_t* stg_w = stg + (warp - 4) * 2 * tc::STG_BYTES;
    uint32_t sc = 0;  // staged chunks (buffer parity)
    int iter = 0;
    GemmWork wk(unit, nunits, num_tiles, ks, num_kb);
    for (; wk.next(); ++iter) {
      const int tile = wk.tile;
      const int tm_ = (opt & 2) ? tile / tiles_n : tile % tiles_m;
      const int tn_ = (opt & 2) ? tile % tiles_n : tile / tiles_m;
      const int m0 = tm_ * C::TILE_M + (int)rank * tc::BM;
      const int n0 = tn_ * BN;
      const int buf = iter & 1;
      const uint32_t aphase = (iter >> 1) & 1;
      const int m = m0 + q * 32 + lane;
      if (num_kb > 0) {
        ptx::mbar_wait(&tfull[buf], aphase);
        ptx::tc_fence_after();
      }
#pragma unroll 1
      for (int c = c_lo; c < c_hi; ++c) {
        float v[32];
        float bvp[32];  // bias prefetch (overlaps the TMEM load)
        bool pre = false;
        if constexpr (ST) {  // ST is only instantiated with EpiStore
          pre = epi.bias != nullptr && n0 + c * 32 < N;
          if (pre) epi.load_bias(n0 + c * 32, N, bvp);
        }
        if (num_kb > 0) {
          ptx::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + buf * BN + c * 32, v);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        }
        if constexpr (ST) {
          const int nc = n0 + c * 32, mw = m0 + q * 32;
          if (nc < N && mw < M) {
            float x[32];
            epi.compute(m, nc, v, M, N, x, pre ? bvp : nullptr);
            // fp32 rows: 2 x 4 KB buffers; bf16 rows (2 KB): 4 buffers in the same space
            uint8_t* sb;
            if (epi.c_bf16) {
              sb = stg_w + (sc & 3) * (tc::STG_BYTES / 2);
              if (lane == 0) ptx::bulk_wait_read3();  // the store that used this buffer 4 chunks ago has read it
            } else {
              sb = stg_w + (sc & 1) * tc::STG_BYTES;
              if (lane == 0) ptx::bulk_wait_read1();  // ... 2 chunks ago
            }
            __syncwarp();
            if (epi.c_bf16) {  // 64 B rows, SWIZZLE_64B: 16 B chunk j of row r at j ^ ((r >> 1) & 3)
              uint4* row = (uint4*)(sb + lane * 64);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                __align__(16) bf16 t8[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) t8[u] = __float2bfloat16_rn(x[j * 8 + u]);
                row[j ^ ((lane >> 1) & 3)] = *(uint4*)t8;
              }
            } else {  // 128 B rows, SWIZZLE_128B: chunk j of row r at j ^ (r & 7)
              float4* row = (float4*)(sb + lane * 128);
#pragma unroll
              for (int j = 0; j < 8; ++j) row[j ^ (lane & 7)] = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (epi.beta || ks != 1) ptx::tma_reduce_add_2d(&tmC, sb, nc, mw);
              else ptx::tma_store_2d(&tmC, sb, nc, mw);
              ptx::bulk_commit();
            }
            ++sc;
          }
        } else {
          if (m < M && n0 + c * 32 < N) epi.apply(m, n0 + c * 32, v, M, N);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0 && num_kb > 0) {
        if constexpr (CG == 2) ptx::mbar_arrive_remote_relaxed(tempty_leader0 + buf * 8);
        else ptx::mbar_arrive_relaxed(&tempty[buf]);
      }
    }
    if constexpr (ST) {
      if (lane == 0) ptx::bulk_wait_all();
    }
  }
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync_all();
  else __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    if constexpr (CG == 2) ptx::tmem_dealloc_cg2(tmem_base, C::TMEM_COLS);
    else ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// fp32 SIMT GEMM (validation mode), same epilogues.
// ---------------------------------------------------------------------------
template <class Epi, typename TI = float>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const TI* __restrict__ A, long long lda, int a_mn,
                                                        const TI* __restrict__ B, long long ldb, int b_mn, int M,
                                                        int N, int K, Epi epi) {
  __shared__ float As[16][65];
  __shared__ float Bs[16][65];
  __shared__ float Cs[64][65];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = tid; i < 16 * 64; i += 256) {
      int kk, r;
      if (a_mn) { kk = i / 64; r = i % 64; } else { r = i / 16; kk = i % 16; }
      int m = m0 + r, k = k0 + kk;
      float va = 0.f;
      if (m < M && k < K) va = to_f<TI>(a_mn ? A[(long long)k * lda + m] : A[(long long)m * lda + k]);
      As[kk][r] = va;
      if (b_mn) { kk = i / 64; r = i % 64; } else { r = i / 16; kk = i % 16; }
      int n = n0 + r;
      k = k0 + kk;
      float vb = 0.f;
      if (n < N && k < K) vb = to_f<TI>(b_mn ? B[(long long)k * ldb + n] : B[(long long)n * ldb + k]);
      Bs[kk][r] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Cs[ty + 16 * i][tx + 16 * j] = acc[i][j];
  __syncthreads();
  if (tid < 128) {
    int r = tid >> 1, ch = tid & 1;
    int m = m0 + r, n = n0 + ch * 32;
    if (m < M && n < N) {
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = Cs[r][ch * 32 + j];
      epi.apply(m, n, v, M, N);
    }
  }
}

}  // namespace cmt
