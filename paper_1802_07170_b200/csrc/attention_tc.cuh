// Luong attention core on tcgen05 (bf16 production mode; attention.py:46-84,
// 139-173, layers.py:183-215).  Every product of the core is a per-sentence
// matrix product, so it runs as a BATCHED tcgen05 GEMM — one work unit per
// (sentence b, output tile) — whose operands are read in place by 3-D TMA maps
// over the token-major activations (row t*B + b of a [T*B][H] matrix is
// element (h, b, t) of a {H, B, T} tensor), with a softmax kernel between:
//
//   forward   scores_b = U_b Hs_b^T          [T x S], K = H   (attention.py:46-54)
//             alpha_b  = masked softmax_s     (layers.py:190-208; masked -> exactly 0)
//             C_b      = alpha_b Hs_b        [T x H], K = S   (attention.py:67-75)
//   backward  dalpha_b = dC_b Hs_b^T         [T x S], K = H   (attention.py:78-84)
//             dsc_b    = alpha (dalpha - sum_s alpha dalpha)  (layers.py:211-215)
//             dU_b     = dsc_b Hs_b          [T x H], K = S   (attention.py:56-64)
//             dHs_b    = alpha_b^T dC_b + dsc_b^T U_b  [S x H], K = T
//
// alpha and dsc are staged as bf16 [B][T][S8] (S8 = S rounded up to 8 for
// 16-byte rows); the same bytes are the K-major A operand of the [T x H]
// products and the MN-major A operand of the [S x H] one.  Out-of-range rows
// and K columns are zero-filled by TMA, so the padding adds exact zeros.
#pragma once
#include "kernels.cuh"
#include "ptx.cuh"

namespace cmt {
namespace bat {
constexpr int BM = 128, BK = 64;
constexpr int THREADS = 256;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-7 epilogue
template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE > 6 ? 6 : (200 * 1024) / STAGE;
  static constexpr int TMEM_COLS = 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 512;
};
}  // namespace bat

// Output of a batched GEMM: C_b[m][n] at C + b*bstride + m*ldc + n (elements),
// fp32 (beta: accumulate) or bf16.
struct BatStore {
  void* C;
  long long ldc, bstride;
  int c_bf16, beta;
};

// One operand's 3-D map: dim0 is the contiguous one (K for K-major, M/N for
// MN-major); bpos = 1: dims {dim0, batch, rows}, 2: {dim0, rows, batch}.
CMT_D void bat_load(const CUtensorMap* tm, uint64_t* bar, void* dst, int c0, int row, int b, int bpos) {
  if (bpos == 1) ptx::tma_load_3d(tm, bar, dst, c0, b, row);
  else ptx::tma_load_3d(tm, bar, dst, c0, row, b);
}

template <int BN, int A_MN, int B_MN>
__global__ void __launch_bounds__(bat::THREADS, 1)
    gemm_bat_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                    int K, int nbatch, int a_bpos, int b_bpos, BatStore epi) {
  using C = bat::Cfg<BN>;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * C::A_BYTES;
  uint64_t* full = (uint64_t*)(smem + S * C::STAGE);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (M + bat::BM - 1) / bat::BM, tiles_n = (N + BN - 1) / BN;
  const int per_b = tiles_m * tiles_n, num_tiles = nbatch * per_b;
  const int num_kb = (K + bat::BK - 1) / bat::BK;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int b = tile / per_b, r = tile % per_b;
        const int m0 = (r % tiles_m) * bat::BM, n0 = (r / tiles_m) * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * C::A_BYTES;
          uint8_t* bb = sB + stage * C::B_BYTES;
          const int k0 = kb * bat::BK;
          if (A_MN) {  // two [64 k][64 m] boxes
            bat_load(&tmA, &full[stage], a, m0, k0, b, a_bpos);
            bat_load(&tmA, &full[stage], a + 64 * bat::BK * 2, m0 + 64, k0, b, a_bpos);
          } else {  // one [128 m][64 k] box
            bat_load(&tmA, &full[stage], a, k0, m0, b, a_bpos);
          }
          if (B_MN) {
#pragma unroll
            for (int q = 0; q < BN / 64; ++q)
              bat_load(&tmB, &full[stage], bb + q * 64 * bat::BK * 2, n0 + q * 64, k0, b, b_bpos);
          } else {
            bat_load(&tmB, &full[stage], bb, k0, n0, b, b_bpos);
          }
          ptx::mbar_expect_tx(&full[stage], C::STAGE);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer =====
      const uint32_t idesc = ptx::idesc_bf16(bat::BM, BN, A_MN, B_MN);
      int stage = 0, iter = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++iter) {
        const int buf = iter & 1;
        ptx::mbar_wait(&tempty[buf], ((iter >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t dtm = tmem_base + buf * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = ptx::smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < bat::BK / 16; ++kk) {
            const uint64_t ad = A_MN ? ptx::smem_desc_sw128(a_addr + kk * 2048, 64 * bat::BK * 2, 1024)
                                     : ptx::smem_desc_sw128(a_addr + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? ptx::smem_desc_sw128(b_addr + kk * 2048, 64 * bat::BK * 2, 1024)
                                     : ptx::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
            ptx::umma_bf16(dtm, ad, bd, idesc, (kb | kk) ? 1u : 0u);
          }
          ptx::umma_commit(&empty[stage]);
          if (kb == num_kb - 1) ptx::umma_commit(&tfull[buf]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {  // ===== epilogue: warp w drains TMEM lanes 32(w-4).. =====
    const int q = warp & 3;
    int iter = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++iter) {
      const int b = tile / per_b, r = tile % per_b;
      const int m0 = (r % tiles_m) * bat::BM, n0 = (r / tiles_m) * BN;
      const int buf = iter & 1;
      ptx::mbar_wait(&tfull[buf], (iter >> 1) & 1);
      ptx::tc_fence_after();
      const int m = m0 + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        ptx::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + buf * BN + c * 32, v);
        const int n = n0 + c * 32;
        if (m >= M || n >= N) continue;
        const long long off = (long long)b * epi.bstride + (long long)m * epi.ldc + n;
        const int nn = min(32, N - n);
        if (epi.c_bf16) {
          bf16* cp = (bf16*)epi.C + off;
          if (nn == 32 && ((((uintptr_t)cp) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              __align__(16) bf16 t8[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) t8[u] = __float2bfloat16_rn(v[j * 8 + u]);
              *(uint4*)(cp + j * 8) = *(uint4*)t8;
            }
          } else {
            for (int j = 0; j < nn; ++j) cp[j] = __float2bfloat16_rn(v[j]);
          }
        } else {
          float* cp = (float*)epi.C + off;
          if (nn == 32 && ((((uintptr_t)cp) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 o = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              if (epi.beta) {
                const float4 p = *(const float4*)(cp + 4 * j);
                o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
              }
              *(float4*)(cp + 4 * j) = o;
            }
          } else {
            for (int j = 0; j < nn; ++j) cp[j] = epi.beta ? cp[j] + v[j] : v[j];
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_relaxed(&tempty[buf]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// Masked column softmax of one (b, t) row per warp (layers.py:190-208):
// alpha[b][t][s] = exp(sc - max) / sum over the unmasked s; masked s exactly 0
// (predicate; the reference's additive -1e9 underflows exp to 0 as well).
// Writes fp32 alpha (the backward's operand) and the bf16 copy [B][T][S8].
__global__ void att_softmax_fwd_kernel(const float* __restrict__ sc, const float* __restrict__ src_mask, int S,
                                       int T, int B, int S8, float* __restrict__ alpha, bf16* __restrict__ a16,
                                       int* __restrict__ status) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= B * T) return;
  const int b = row / T;
  const float* x = sc + (long long)row * S;
  float mx = -INFINITY;
  bool bad = false;
  for (int s = lane; s < S; s += 32) {
    const float v = x[s];
    bad |= !isfinite(v);
    if (src_mask[(long long)s * B + b] != 0.f) mx = fmaxf(mx, v);
  }
  mx = warp_max(mx);
  float z = 0.f;
  for (int s = lane; s < S; s += 32)
    if (src_mask[(long long)s * B + b] != 0.f) z += expf(x[s] - mx);
  z = warp_sum(z);
  for (int s = lane; s < S8; s += 32) {
    const float a = (s < S && src_mask[(long long)s * B + b] != 0.f) ? expf(x[s] - mx) / z : 0.f;
    if (s < S) alpha[(long long)row * S + s] = a;
    a16[(long long)row * S8 + s] = __float2bfloat16_rn(a);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_SCORES);
}

// Softmax backward of one (b, t) row per warp (layers.py:211-215):
// dsc = alpha (dalpha - sum_s alpha dalpha), as bf16 [B][T][S8].
__global__ void att_softmax_bwd_kernel(const float* __restrict__ alpha, const float* __restrict__ dal, int S, int T,
                                       int B, int S8, bf16* __restrict__ d16) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= B * T) return;
  const float* a = alpha + (long long)row * S;
  const float* g = dal + (long long)row * S;
  float dot = 0.f;
  for (int s = lane; s < S; s += 32) dot = fmaf(a[s], g[s], dot);
  dot = warp_sum(dot);
  for (int s = lane; s < S8; s += 32) d16[(long long)row * S8 + s] = __float2bfloat16_rn(s < S ? a[s] * (g[s] - dot) : 0.f);
}

}  // namespace cmt
