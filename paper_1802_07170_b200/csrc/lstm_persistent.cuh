// Persistent recurrent LSTM kernels (bf16 production path).
//
// One cooperative launch runs a whole scan (all timesteps of one layer /
// direction).  CTA g owns a slice of W_h that stays resident in shared memory
// for the entire scan; each step it streams the previous step's h_{t-1}
// (forward) or dU_{t+1} (backward) for the whole batch through a TMA ring,
// issues tcgen05.mma into TMEM, and runs the fused cell epilogue with the
// recurrent state (c, h / dh, dc carries) held in registers of the thread that
// owns (batch row, units).  Steps are separated by a grid-wide release/acquire
// counter instead of kernel launches.  Reference semantics: layers.py:344-395
// (cell forward/backward), layers.py:440-493 (masked scan / BPTT).
//
//   forward : CTA g owns gate columns [64g, 64g+64) = units [16g, 16g+16);
//             acc[b][gc] = sum_j h_{t-1}[b][j] W[din+j][gc]   (M=B<=128, N=64, K=H)
//   backward: CTA g owns units [16g, 16g+16);
//             acc[b][j]  = sum_gc dU_{t+1}[b][gc] W[din+j][gc] (M=B<=128, N=16, K=4H)
#pragma once
#include "ptx.cuh"

namespace cmt {
namespace pr {
constexpr int THREADS = 256;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-7 cell epilogue
constexpr int MAX_STAGES = 8;
constexpr int ROWS = 64;               // batch rows per CTA (the other 64 accumulator rows are don't-care)
constexpr int KBLK = ROWS * 128;       // one k-block tile in smem: [64 rows][64 cols] bf16 = 8 KB
constexpr int KBOX = 4;                // k-blocks fetched per (3-D) TMA instruction = one pipeline stage
constexpr int STAGE_BYTES = KBOX * KBLK;
constexpr int PAD = KBLK;              // UMMA M=128 reads 128 rows: the last tile spills 8 KB past its stage
constexpr int FWD_NG = 64;             // gate columns per CTA
constexpr int BWD_NU = 16;             // units per CTA
constexpr size_t SMEM_LIMIT = 227 * 1024;
// as many TMA stages as fit beside the resident W_h slice (H*128 bytes)
inline int stages_for(int H) {
  long long room = (long long)SMEM_LIMIT - 1024 - 256 - PAD - (long long)H * 128;
  long long s = room / STAGE_BYTES;
  return (int)(s > MAX_STAGES ? MAX_STAGES : s);
}
inline size_t smem_bytes(int H) {
  return 1024 + (size_t)H * 128 + (size_t)stages_for(H) * STAGE_BYTES + PAD + 256;
}
}  // namespace pr

struct LstmFwdP {
  const float* ux;      // [steps*B][4H] (bias folded)
  bf16* y;              // y view: h_t at rows t*B+b
  const bf16* hprev;    // h_{t-1} view (initial state read at the first step)
  float* cst;           // c view
  const float* cprev;   // c_{t-1} view
  float* acts;          // [steps*B][4H]
  float* tcache;        // [steps*B][H]
  const float* mask;    // [steps][B] or null
  unsigned* flag;       // zeroed before launch
  int steps, B, H, din, reverse;
  int hrow0;            // row of h_{-1}(t=0) in the Yext tensor map
  int stages;
  unsigned long long* trace;  // debug: per-step phase timestamps of CTA 0 (or null)
};
CMT_D unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(pr::THREADS, 1)
    lstm_fwd_persistent(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW, LstmFwdP p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int KB = p.H / 64;
  uint8_t* sW = smem;                     // KB x [64 K rows][64 N] (MN-major atoms)
  uint8_t* sA = smem + (size_t)KB * 8192;  // stages x KBOX x [64 rows][64] (K-major) + pad
  uint64_t* full = (uint64_t*)(sA + p.stages * pr::STAGE_BYTES + pr::PAD);
  uint64_t* empty = full + pr::MAX_STAGES;
  uint64_t* wfull = empty + pr::MAX_STAGES;
  uint64_t* tfull = wfull + 1;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int nh = (p.B + pr::ROWS - 1) / pr::ROWS;
  const int half = blockIdx.x % nh;
  const int n0 = (blockIdx.x / nh) * pr::FWD_NG;
  const int u0 = n0 >> 2;
  const int r0 = half * pr::ROWS;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tmH);
    ptx::prefetch_tmap(&tmW);
    for (int i = 0; i < p.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(wfull, 1);
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty, 2);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 64);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_expect_tx(wfull, KB * 8192);
      for (int kb = 0; kb < KB; ++kb) ptx::tma_load_2d(&tmW, wfull, sW + kb * 8192, n0, p.din + kb * 64);
      int stage = 0;
      uint32_t phase = 0;
      for (int s = 0; s < p.steps; ++s) {
        const int t = p.reverse ? p.steps - 1 - s : s;
        if (s > 0) {
          const unsigned target = (unsigned)(G * s);
          while (ptx::ld_relaxed(p.flag) < target) {}
          ptx::fence_acquire_gpu();
          ptx::fence_proxy_async_global();
        }
        if (p.trace && blockIdx.x == 0) p.trace[s * 8 + 0] = gtimer();
        const int hrow = p.hrow0 + t * p.B + r0;
        for (int kb = 0; kb < KB; kb += pr::KBOX) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::tma_load_3d(&tmH, &full[stage], sA + stage * pr::STAGE_BYTES, 0, hrow, kb);
          ptx::mbar_expect_tx(&full[stage], pr::STAGE_BYTES);
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, pr::FWD_NG, 0, 1);
      ptx::mbar_wait(wfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t wbase = ptx::smem_u32(sW);
      for (int s = 0; s < p.steps; ++s) {
        ptx::mbar_wait(tempty, (s & 1) ^ 1);
        ptx::tc_fence_after();
        for (int kb0 = 0; kb0 < KB; kb0 += pr::KBOX) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (p.trace && blockIdx.x == 0 && (kb0 == 0 || kb0 == KB - pr::KBOX))
            p.trace[s * 8 + 4 + (kb0 == 0 ? 0 : 3)] = gtimer();
          const uint32_t a0 = ptx::smem_u32(sA + stage * pr::STAGE_BYTES);
#pragma unroll
          for (int j = 0; j < pr::KBOX; ++j) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint64_t ad = ptx::smem_desc_sw128(a0 + j * pr::KBLK + kk * 32, 16, 1024);
              uint64_t bd = ptx::smem_desc_sw128(wbase + (kb0 + j) * 8192 + kk * 2048, 8192, 1024);
              ptx::umma_bf16(tmem, ad, bd, idesc, (kb0 | j | kk) ? 1u : 0u);
            }
          }
          ptx::umma_commit(&empty[stage]);
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(tfull);
      }
    }
  } else if (warp >= 4 && warp < 6) {
    const int q = warp & 3;
    const int b = r0 + q * 32 + lane;
    const bool valid = b < p.B && b < r0 + pr::ROWS;
    const long long H = p.H;
    float c[16], h[16];
    {
      const int t0 = p.reverse ? p.steps - 1 : 0;
      const long long r0 = (long long)t0 * p.B + b;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        c[u] = valid ? p.cprev[r0 * H + u0 + u] : 0.f;
        h[u] = valid ? __bfloat162float(p.hprev[r0 * H + u0 + u]) : 0.f;
      }
    }
    for (int s = 0; s < p.steps; ++s) {
      const int t = p.reverse ? p.steps - 1 - s : s;
      const long long row = (long long)t * p.B + b;
      // prefetch this step's inputs before waiting for the accumulator
      float4 x[16];
      float mk = 1.f;
      if (valid) {
        const float4* uxr = (const float4*)(p.ux + row * 4 * H + n0);
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = __ldg(uxr + u);
        if (p.mask) mk = __ldg(p.mask + row);
      }
      ptx::mbar_wait(tfull, s & 1);
      ptx::tc_fence_after();
      if (p.trace && blockIdx.x == 0 && threadIdx.x == 128) p.trace[s * 8 + 1] = gtimer();
      float v[64];
      ptx::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16), v);
      ptx::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + 32, v + 32);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(tempty);
      float tcv[16];
      if (valid) {
        __align__(16) bf16 hb[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float gi = ptx::sigmoid_fast(v[4 * u + 0] + x[u].x);
          const float gf = ptx::sigmoid_fast(v[4 * u + 1] + x[u].y);
          const float gg = ptx::tanh_fast(v[4 * u + 2] + x[u].z);
          const float go = ptx::sigmoid_fast(v[4 * u + 3] + x[u].w);
          const float cn = gf * c[u] + gi * gg;
          const float tcn = ptx::tanh_fast(cn);
          const float hn = go * tcn;
          if (p.mask) {
            h[u] = mk * hn + (1.f - mk) * h[u];
            c[u] = mk * cn + (1.f - mk) * c[u];
          } else {
            h[u] = hn;
            c[u] = cn;
          }
          x[u] = make_float4(gi, gf, gg, go);  // reuse: activations for the cache
          tcv[u] = tcn;
          hb[u] = __float2bfloat16_rn(h[u]);
        }
        uint4* yr = (uint4*)(p.y + row * H + u0);
        yr[0] = ((uint4*)hb)[0];
        yr[1] = ((uint4*)hb)[1];
      }
      if (p.trace && blockIdx.x == 0 && threadIdx.x == 128) p.trace[s * 8 + 2] = gtimer();
      // publish h_t (the only value other CTAs need), then write the BPTT caches
      ptx::named_bar_sync(1, 64);
      if (threadIdx.x == 128) {
        ptx::red_release_add(p.flag, 1u);
        if (p.trace && blockIdx.x == 0) p.trace[s * 8 + 3] = gtimer();
      }
      if (valid) {
        float4* ar = (float4*)(p.acts + row * 4 * H + n0);
#pragma unroll
        for (int u = 0; u < 16; ++u) ar[u] = x[u];
        float4* tcr = (float4*)(p.tcache + row * H + u0);
        float4* csr = (float4*)(p.cst + row * H + u0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          tcr[k] = make_float4(tcv[4 * k], tcv[4 * k + 1], tcv[4 * k + 2], tcv[4 * k + 3]);
          csr[k] = make_float4(c[4 * k], c[4 * k + 1], c[4 * k + 2], c[4 * k + 3]);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 64);
  }
}

struct LstmBwdP {
  const float* dy;       // [steps*B][H]
  const float* acts;     // [steps*B][4H]
  const float* tcache;   // [steps*B][H]
  const float* cprev;    // c_{t-1} view, rows t*B+b
  const float* mask;     // [steps][B] or null
  bf16* dU;              // [steps*B][4H]
  const float* dh_final; // [B][H] or null
  const float* dc_final;
  float* dh0;            // [B][H] or null: grads of the initial state
  float* dc0;
  unsigned* flag;
  int steps, B, H, din, reverse;
  int stages;
  unsigned long long* trace;
};

__global__ void __launch_bounds__(pr::THREADS, 1)
    lstm_bwd_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, LstmBwdP p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int KB = p.H / 16;                 // 4H / 64 k-blocks
  uint8_t* sW = smem;                      // KB x [16 rows][64 K] (K-major), 2 KB each
  uint8_t* sA = smem + (size_t)KB * 2048;  // stages x KBOX x [64 rows][64] + pad
  uint64_t* full = (uint64_t*)(sA + p.stages * pr::STAGE_BYTES + pr::PAD);
  uint64_t* empty = full + pr::MAX_STAGES;
  uint64_t* wfull = empty + pr::MAX_STAGES;
  uint64_t* tfull = wfull + 1;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int nh = (p.B + pr::ROWS - 1) / pr::ROWS;
  const int half = blockIdx.x % nh;
  const int u0 = (blockIdx.x / nh) * pr::BWD_NU;
  const int r0 = half * pr::ROWS;
  const int rounds = p.steps + (p.dh0 ? 1 : 0);
  auto time_of = [&](int pos) { return p.reverse ? p.steps - 1 - pos : pos; };
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmW);
    for (int i = 0; i < p.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(wfull, 1);
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty, 2);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 32);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_expect_tx(wfull, KB * 2048);
      for (int kb = 0; kb < KB; ++kb) ptx::tma_load_2d(&tmW, wfull, sW + kb * 2048, kb * 64, p.din + u0);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 1; i < rounds; ++i) {
        // round i consumes dU of the position finished in round i-1
        const unsigned target = (unsigned)(G * i);
        while (ptx::ld_relaxed(p.flag) < target) {}
          ptx::fence_acquire_gpu();
        ptx::fence_proxy_async_global();
        const int arow = time_of(p.steps - i) * p.B + r0;
        for (int kb = 0; kb < KB; kb += pr::KBOX) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::tma_load_3d(&tmA, &full[stage], sA + stage * pr::STAGE_BYTES, 0, arow, kb);
          ptx::mbar_expect_tx(&full[stage], pr::STAGE_BYTES);
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, pr::BWD_NU, 0, 0);
      ptx::mbar_wait(wfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t wbase = ptx::smem_u32(sW);
      for (int i = 1; i < rounds; ++i) {
        ptx::mbar_wait(tempty, ((i - 1) & 1) ^ 1);
        ptx::tc_fence_after();
        for (int kb0 = 0; kb0 < KB; kb0 += pr::KBOX) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a0 = ptx::smem_u32(sA + stage * pr::STAGE_BYTES);
#pragma unroll
          for (int j = 0; j < pr::KBOX; ++j) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint64_t ad = ptx::smem_desc_sw128(a0 + j * pr::KBLK + kk * 32, 16, 1024);
              uint64_t bd = ptx::smem_desc_sw128(wbase + (kb0 + j) * 2048 + kk * 32, 16, 1024);
              ptx::umma_bf16(tmem, ad, bd, idesc, (kb0 | j | kk) ? 1u : 0u);
            }
          }
          ptx::umma_commit(&empty[stage]);
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(tfull);
      }
    }
  } else if (warp >= 4 && warp < 6) {
    const int q = warp & 3;
    const int b = r0 + q * 32 + lane;
    const bool valid = b < p.B && b < r0 + pr::ROWS;
    const long long H = p.H;
    float dhc[16], dc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      dhc[u] = (valid && p.dh_final) ? p.dh_final[(long long)b * H + u0 + u] : 0.f;
      dc[u] = (valid && p.dc_final) ? p.dc_final[(long long)b * H + u0 + u] : 0.f;
    }
    for (int i = 0; i < rounds; ++i) {
      const bool cell = i < p.steps;
      const int t = cell ? time_of(p.steps - 1 - i) : 0;
      const long long row = (long long)t * p.B + b;
      // prefetch the cell inputs of this round before waiting for the accumulator
      float4 dy4[4], tc4[4], cp4[4], a4[16];
      float mk = 1.f;
      if (valid && cell) {
        const float4* dyr = (const float4*)(p.dy + row * H + u0);
        const float4* tcr = (const float4*)(p.tcache + row * H + u0);
        const float4* cpr = (const float4*)(p.cprev + row * H + u0);
        const float4* ar = (const float4*)(p.acts + row * 4 * H + 4 * u0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          dy4[k] = __ldg(dyr + k);
          tc4[k] = __ldg(tcr + k);
          cp4[k] = __ldg(cpr + k);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) a4[u] = __ldg(ar + u);
        if (p.mask) mk = __ldg(p.mask + row);
      }
      float acc[16];
      if (i > 0) {
        ptx::mbar_wait(tfull, (i - 1) & 1);
        ptx::tc_fence_after();
        ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16), acc);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tempty);
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) acc[u] = 0.f;
      }
      if (valid) {
        if (cell) {
          __align__(16) bf16 du[64];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float dyv[4] = {dy4[k].x, dy4[k].y, dy4[k].z, dy4[k].w};
            const float tcv[4] = {tc4[k].x, tc4[k].y, tc4[k].z, tc4[k].w};
            const float cpv[4] = {cp4[k].x, cp4[k].y, cp4[k].z, cp4[k].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int u = 4 * k + e;
              const float dh = acc[u] + dhc[u] + dyv[e];
              float dhn = dh, dcn = dc[u], dhcar = 0.f, dccar = 0.f;
              if (p.mask) {
                dhn = mk * dh; dcn = mk * dc[u];
                dhcar = (1.f - mk) * dh; dccar = (1.f - mk) * dc[u];
              }
              const float4 a = a4[u];  // i f g o
              const float tc = tcv[e];
              const float dct = dhn * a.w * (1.f - tc * tc) + dcn;
              du[4 * u + 0] = __float2bfloat16_rn(dct * a.z * (a.x * (1.f - a.x)));
              du[4 * u + 1] = __float2bfloat16_rn(dct * cpv[e] * (a.y * (1.f - a.y)));
              du[4 * u + 2] = __float2bfloat16_rn(dct * a.x * (1.f - a.z * a.z));
              du[4 * u + 3] = __float2bfloat16_rn(dhn * tc * (a.w * (1.f - a.w)));
              dc[u] = dct * a.y + dccar;
              dhc[u] = dhcar;
            }
          }
          uint4* dur = (uint4*)(p.dU + row * 4 * H + 4 * u0);
#pragma unroll
          for (int k = 0; k < 8; ++k) dur[k] = ((uint4*)du)[k];
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            p.dh0[(long long)b * H + u0 + u] = acc[u] + dhc[u];
            p.dc0[(long long)b * H + u0 + u] = dc[u];
          }
        }
      }
      ptx::named_bar_sync(1, 64);
      if (threadIdx.x == 128) ptx::red_release_add(p.flag, 1u);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 32);
  }
}

}  // namespace cmt
