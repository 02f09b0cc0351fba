// Cluster-split persistent recurrent LSTM kernels (bf16 production path).
//
// Same contract as lstm_persistent.cuh (one cooperative launch per scan,
// W_h resident in smem, register-held recurrent state, grid step barrier), but
// the recurrent contraction of each column group is split over the CTAs of a
// thread-block cluster (K-split).  Each CTA then holds only 1/KS of the W_h
// slice, so its smem fits enough 32 KB TMA stages for the whole per-step
// operand stream to be in flight at once; the partial accumulators are summed
// through distributed shared memory (st.shared::cluster + a remote mbarrier
// arrive) and every CTA runs the cell update for 1/KS of the group's units.
//
//   forward  (KS=2): cluster owns 64 gate columns (16 units), CTA rank r
//            contracts h_{t-1}[:, r*H/2 : (r+1)*H/2]; cell for units 8r..8r+7
//   backward (KS=4): cluster owns 32 units, CTA rank r contracts dU over gate
//            columns [r*H, (r+1)*H); cell backward for units 8r..8r+7
// Reference semantics: layers.py:344-395, 440-493.
#pragma once
#include "lstm_persistent.cuh"

namespace cmt {
namespace cl {
constexpr int THREADS = 256;
constexpr int ROWS = 128;             // whole batch per CTA (B <= 128)
constexpr int KBOX = 2;               // k-blocks per 3-D TMA = one 32 KB stage
constexpr int KBLK = ROWS * 128;      // [128 rows][64] bf16 = 16 KB
constexpr int STAGE_BYTES = KBOX * KBLK;
constexpr int MAX_STAGES = 8;
constexpr int FWD_KS = 2, FWD_NG = 64;  // gate columns per cluster
constexpr int BWD_KS = 4, BWD_NU = 32;  // units per cluster
constexpr int UPC = 8;                  // units per CTA in the cell epilogue
constexpr size_t SMEM_LIMIT = 227 * 1024;
inline size_t fwd_w_bytes(int H) { return (size_t)(H / FWD_KS / 64) * 8192; }        // [64 K][64 gc] per k-block
inline size_t bwd_w_bytes(int H) { return (size_t)(H / 64) * (BWD_NU * 128); }       // [32 rows][64] per k-block
constexpr size_t FWD_X = ROWS * 32 * 4;                                              // partner half: [128][32] f32
constexpr size_t BWD_X = BWD_KS * ROWS * UPC * 4;                                    // [4 senders][128][8] f32
inline int stages_for(size_t fixed) {
  long long room = (long long)SMEM_LIMIT - 1024 - 256 - (long long)fixed;
  long long s = room / STAGE_BYTES;
  return (int)(s > MAX_STAGES ? MAX_STAGES : s);
}
inline int fwd_stages(int H) { return stages_for(fwd_w_bytes(H) + FWD_X); }
inline int bwd_stages(int H) { return stages_for(bwd_w_bytes(H) + BWD_X); }
inline size_t fwd_smem(int H) { return 1024 + fwd_w_bytes(H) + FWD_X + (size_t)fwd_stages(H) * STAGE_BYTES + 256; }
inline size_t bwd_smem(int H) { return 1024 + bwd_w_bytes(H) + BWD_X + (size_t)bwd_stages(H) * STAGE_BYTES + 256; }
}  // namespace cl

__global__ void __launch_bounds__(cl::THREADS, 1)
    lstm_fwd_cluster(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW, LstmFwdP p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int KBL = p.H / 64 / cl::FWD_KS;  // k-blocks contracted by this CTA
  uint8_t* sW = smem;
  float* xbuf = (float*)(sW + (size_t)KBL * 8192);
  uint8_t* sA = (uint8_t*)xbuf + cl::FWD_X;
  uint64_t* full = (uint64_t*)(sA + (size_t)p.stages * cl::STAGE_BYTES);
  uint64_t* empty = full + cl::MAX_STAGES;
  uint64_t* wfull = empty + cl::MAX_STAGES;
  uint64_t* tfull = wfull + 1;
  uint64_t* tempty = tfull + 1;
  uint64_t* xfull = tempty + 1;
  uint32_t* tmem_slot = (uint32_t*)(xfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const uint32_t r = ptx::cluster_rank();
  const uint32_t partner = r ^ 1u;
  const int n0 = (blockIdx.x / cl::FWD_KS) * cl::FWD_NG;  // group gate columns
  const int kb_base = (int)r * KBL;                        // first k-block of this CTA's K range
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tmH);
    ptx::prefetch_tmap(&tmW);
    for (int i = 0; i < p.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(wfull, 1);
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty, 4);
    ptx::mbar_init(xfull, 4);  // the partner's 4 epilogue warps
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 64);
  ptx::tc_fence_before();
  ptx::cluster_sync_all();  // barrier inits visible cluster-wide before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_expect_tx(wfull, KBL * 8192);
      for (int kb = 0; kb < KBL; ++kb)
        ptx::tma_load_2d(&tmW, wfull, sW + kb * 8192, n0, p.din + (kb_base + kb) * 64);
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
        const int hrow = p.hrow0 + t * p.B;
        for (int kb = 0; kb < KBL; kb += cl::KBOX) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::tma_load_3d(&tmH, &full[stage], sA + stage * cl::STAGE_BYTES, 0, hrow, kb_base + kb);
          ptx::mbar_expect_tx(&full[stage], cl::STAGE_BYTES);
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, cl::FWD_NG, 0, 1);
      ptx::mbar_wait(wfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t wbase = ptx::smem_u32(sW);
      for (int s = 0; s < p.steps; ++s) {
        ptx::mbar_wait(tempty, (s & 1) ^ 1);
        ptx::tc_fence_after();
        for (int kb0 = 0; kb0 < KBL; kb0 += cl::KBOX) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a0 = ptx::smem_u32(sA + stage * cl::STAGE_BYTES);
#pragma unroll
          for (int j = 0; j < cl::KBOX; ++j) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint64_t ad = ptx::smem_desc_sw128(a0 + j * cl::KBLK + kk * 32, 16, 1024);
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
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int b = q * 32 + lane;
    const bool valid = b < p.B;
    const long long H = p.H;
    const int cm = (int)r * 32;              // my gate columns within the group
    const int cp = (int)partner * 32;        // partner's
    const int u0 = (n0 + cm) >> 2;           // my first unit
    const uint32_t x_remote = ptx::mapa(ptx::smem_u32(xbuf + b * 32), partner);
    const uint32_t xfull_remote = ptx::mapa(ptx::smem_u32(xfull), partner);
    float c[cl::UPC], h[cl::UPC];
    {
      const int t0 = p.reverse ? p.steps - 1 : 0;
      const long long r0 = (long long)t0 * p.B + b;
#pragma unroll
      for (int u = 0; u < cl::UPC; ++u) {
        c[u] = valid ? p.cprev[r0 * H + u0 + u] : 0.f;
        h[u] = valid ? __bfloat162float(p.hprev[r0 * H + u0 + u]) : 0.f;
      }
    }
    for (int s = 0; s < p.steps; ++s) {
      const int t = p.reverse ? p.steps - 1 - s : s;
      const long long row = (long long)t * p.B + b;
      float4 x[cl::UPC];
      float mk = 1.f;
      if (valid) {
        const float4* uxr = (const float4*)(p.ux + row * 4 * H + n0 + cm);
#pragma unroll
        for (int u = 0; u < cl::UPC; ++u) x[u] = __ldg(uxr + u);
        if (p.mask) mk = __ldg(p.mask + row);
      }
      ptx::mbar_wait(tfull, s & 1);
      ptx::tc_fence_after();
      if (p.trace && blockIdx.x == 0 && threadIdx.x == 128) p.trace[s * 8 + 1] = gtimer();
      float v[32], w[32];
      const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
      ptx::tmem_ld32(tl + cp, v);
      ptx::tmem_ld32(tl + cm, w);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(tempty);
      // partner's K-half contribution to ITS units -> partner's smem
#pragma unroll
      for (int k = 0; k < 8; ++k) ptx::st_cluster_v4(x_remote + k * 16, v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
      ptx::fence_acq_rel_cluster();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_remote(xfull_remote);
      ptx::mbar_wait_cluster(xfull, s & 1);
      const float4* xr = (const float4*)(xbuf + b * 32);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 z = xr[k];
        w[4 * k] += z.x; w[4 * k + 1] += z.y; w[4 * k + 2] += z.z; w[4 * k + 3] += z.w;
      }
      if (p.trace && blockIdx.x == 0 && threadIdx.x == 128) p.trace[s * 8 + 2] = gtimer();
      float tcv[cl::UPC];
      if (valid) {
        __align__(16) bf16 hb[cl::UPC];
#pragma unroll
        for (int u = 0; u < cl::UPC; ++u) {
          const float gi = ptx::sigmoid_fast(w[4 * u + 0] + x[u].x);
          const float gf = ptx::sigmoid_fast(w[4 * u + 1] + x[u].y);
          const float gg = ptx::tanh_fast(w[4 * u + 2] + x[u].z);
          const float go = ptx::sigmoid_fast(w[4 * u + 3] + x[u].w);
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
          x[u] = make_float4(gi, gf, gg, go);
          tcv[u] = tcn;
          hb[u] = __float2bfloat16_rn(h[u]);
        }
        *(uint4*)(p.y + row * H + u0) = *(uint4*)hb;
      }
      ptx::named_bar_sync(1, 128);
      if (threadIdx.x == 128) {
        ptx::red_release_add(p.flag, 1u);
        if (p.trace && blockIdx.x == 0) p.trace[s * 8 + 3] = gtimer();
      }
      if (valid) {
        float4* ar = (float4*)(p.acts + row * 4 * H + n0 + cm);
#pragma unroll
        for (int u = 0; u < cl::UPC; ++u) ar[u] = x[u];
        float4* tcr = (float4*)(p.tcache + row * H + u0);
        float4* csr = (float4*)(p.cst + row * H + u0);
        tcr[0] = make_float4(tcv[0], tcv[1], tcv[2], tcv[3]);
        tcr[1] = make_float4(tcv[4], tcv[5], tcv[6], tcv[7]);
        csr[0] = make_float4(c[0], c[1], c[2], c[3]);
        csr[1] = make_float4(c[4], c[5], c[6], c[7]);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();  // no CTA leaves while its partner may still write its smem
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 64);
  }
}

__global__ void __launch_bounds__(cl::THREADS, 1)
    lstm_bwd_cluster(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, LstmBwdP p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int KBL = p.H / 64;  // k-blocks over this CTA's gate-column range [r*H, (r+1)*H)
  uint8_t* sW = smem;                                   // KBL x [32 rows][64] (K-major)
  float* xbuf = (float*)(sW + (size_t)KBL * (cl::BWD_NU * 128));
  uint8_t* sA = (uint8_t*)xbuf + cl::BWD_X;
  uint64_t* full = (uint64_t*)(sA + (size_t)p.stages * cl::STAGE_BYTES);
  uint64_t* empty = full + cl::MAX_STAGES;
  uint64_t* wfull = empty + cl::MAX_STAGES;
  uint64_t* tfull = wfull + 1;
  uint64_t* tempty = tfull + 1;
  uint64_t* xfull = tempty + 1;
  uint32_t* tmem_slot = (uint32_t*)(xfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const uint32_t r = ptx::cluster_rank();
  const int ug = (blockIdx.x / cl::BWD_KS) * cl::BWD_NU;  // group's first unit
  const int kb_base = (int)r * KBL;                       // gate-column k-block base of this CTA
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
    ptx::mbar_init(tempty, 4);
    ptx::mbar_init(xfull, 1);  // the owner's expect_tx; partner bytes arrive by st.async complete_tx
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 32);
  ptx::tc_fence_before();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_expect_tx(wfull, KBL * cl::BWD_NU * 128);
      for (int kb = 0; kb < KBL; ++kb)
        ptx::tma_load_2d(&tmW, wfull, sW + kb * (cl::BWD_NU * 128), (kb_base + kb) * 64, p.din + ug);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 1; i < rounds; ++i) {
        const unsigned target = (unsigned)(G * i);
        while (ptx::ld_relaxed(p.flag) < target) {}
        ptx::fence_acquire_gpu();
        ptx::fence_proxy_async_global();
        if (p.trace && blockIdx.x == 0) p.trace[i * 8 + 0] = gtimer();
        const int arow = time_of(p.steps - i) * p.B;
        for (int kb = 0; kb < KBL; kb += cl::KBOX) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::tma_load_3d(&tmA, &full[stage], sA + stage * cl::STAGE_BYTES, 0, arow, kb_base + kb);
          ptx::mbar_expect_tx(&full[stage], cl::STAGE_BYTES);
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, cl::BWD_NU, 0, 0);
      ptx::mbar_wait(wfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t wbase = ptx::smem_u32(sW);
      for (int i = 1; i < rounds; ++i) {
        ptx::mbar_wait(tempty, ((i - 1) & 1) ^ 1);
        ptx::tc_fence_after();
        for (int kb0 = 0; kb0 < KBL; kb0 += cl::KBOX) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a0 = ptx::smem_u32(sA + stage * cl::STAGE_BYTES);
#pragma unroll
          for (int j = 0; j < cl::KBOX; ++j) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint64_t ad = ptx::smem_desc_sw128(a0 + j * cl::KBLK + kk * 32, 16, 1024);
              uint64_t bd = ptx::smem_desc_sw128(wbase + (kb0 + j) * (cl::BWD_NU * 128) + kk * 32, 16, 1024);
              ptx::umma_bf16(tmem, ad, bd, idesc, (kb0 | j | kk) ? 1u : 0u);
            }
          }
          ptx::umma_commit(&empty[stage]);
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(tfull);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int b = q * 32 + lane;
    const bool valid = b < p.B;
    const long long H = p.H;
    const int u0 = ug + (int)r * cl::UPC;  // my 8 units
    float dhc[cl::UPC], dc[cl::UPC];
#pragma unroll
    for (int u = 0; u < cl::UPC; ++u) {
      dhc[u] = (valid && p.dh_final) ? p.dh_final[(long long)b * H + u0 + u] : 0.f;
      dc[u] = (valid && p.dc_final) ? p.dc_final[(long long)b * H + u0 + u] : 0.f;
    }
    uint32_t x_remote[cl::BWD_KS], xf_remote[cl::BWD_KS];
#pragma unroll
    for (int pr_ = 0; pr_ < cl::BWD_KS; ++pr_) {
      // my slot in partner pr_'s buffer: xbuf[r][b][0..8)
      x_remote[pr_] = ptx::mapa(ptx::smem_u32(xbuf + ((size_t)r * cl::ROWS + b) * cl::UPC), pr_);
      xf_remote[pr_] = ptx::mapa(ptx::smem_u32(xfull), pr_);
    }
    for (int i = 0; i < rounds; ++i) {
      const bool cell = i < p.steps;
      const int t = cell ? time_of(p.steps - 1 - i) : 0;
      const long long row = (long long)t * p.B + b;
      float4 dy4[2], tc4[2], cp4[2], a4[cl::UPC];
      float mk = 1.f;
      if (valid && cell) {
        const float4* dyr = (const float4*)(p.dy + row * H + u0);
        const float4* tcr = (const float4*)(p.tcache + row * H + u0);
        const float4* cpr = (const float4*)(p.cprev + row * H + u0);
        const float4* ar = (const float4*)(p.acts + row * 4 * H + 4 * u0);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          dy4[k] = __ldg(dyr + k);
          tc4[k] = __ldg(tcr + k);
          cp4[k] = __ldg(cpr + k);
        }
#pragma unroll
        for (int u = 0; u < cl::UPC; ++u) a4[u] = __ldg(ar + u);
        if (p.mask) mk = __ldg(p.mask + row);
      }
      float acc[cl::UPC];
      if (i > 0) {
        ptx::mbar_wait(tfull, (i - 1) & 1);
        ptx::tc_fence_after();
        if (p.trace && blockIdx.x == 0 && threadIdx.x == 128) p.trace[i * 8 + 1] = gtimer();
        float v[32];
        ptx::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16), v);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tempty);
        // send each partner its 8 columns of my partial sum (async remote stores
        // whose bytes complete the partner's xfull phase)
#pragma unroll
        for (int pr_ = 0; pr_ < cl::BWD_KS; ++pr_) {
          if (pr_ == (int)r) continue;
          ptx::st_async_v4(x_remote[pr_], v[8 * pr_], v[8 * pr_ + 1], v[8 * pr_ + 2], v[8 * pr_ + 3], xf_remote[pr_]);
          ptx::st_async_v4(x_remote[pr_] + 16, v[8 * pr_ + 4], v[8 * pr_ + 5], v[8 * pr_ + 6], v[8 * pr_ + 7],
                           xf_remote[pr_]);
        }
        if (threadIdx.x == 128) ptx::mbar_expect_tx(xfull, (cl::BWD_KS - 1) * cl::ROWS * cl::UPC * 4);
#pragma unroll
        for (int u = 0; u < cl::UPC; ++u) acc[u] = v[8 * r + u];
        ptx::mbar_wait_cluster(xfull, (i - 1) & 1);
        if (p.trace && blockIdx.x == 0 && threadIdx.x == 128) p.trace[i * 8 + 2] = gtimer();
#pragma unroll
        for (int pr_ = 0; pr_ < cl::BWD_KS; ++pr_) {
          if (pr_ == (int)r) continue;
          const float4* xr = (const float4*)(xbuf + ((size_t)pr_ * cl::ROWS + b) * cl::UPC);
          const float4 z0 = xr[0], z1 = xr[1];
          acc[0] += z0.x; acc[1] += z0.y; acc[2] += z0.z; acc[3] += z0.w;
          acc[4] += z1.x; acc[5] += z1.y; acc[6] += z1.z; acc[7] += z1.w;
        }
      } else {
#pragma unroll
        for (int u = 0; u < cl::UPC; ++u) acc[u] = 0.f;
      }
      if (valid) {
        if (cell) {
          __align__(16) bf16 du[4 * cl::UPC];
#pragma unroll
          for (int k = 0; k < 2; ++k) {
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
              const float4 a = a4[u];
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
          for (int k = 0; k < 4; ++k) dur[k] = ((uint4*)du)[k];
        } else {
#pragma unroll
          for (int u = 0; u < cl::UPC; ++u) {
            p.dh0[(long long)b * H + u0 + u] = acc[u] + dhc[u];
            p.dc0[(long long)b * H + u0 + u] = dc[u];
          }
        }
      }
      if (p.trace && blockIdx.x == 0 && threadIdx.x == 128) p.trace[i * 8 + 3] = gtimer();
      ptx::named_bar_sync(1, 128);
      if (threadIdx.x == 128) {
        ptx::red_release_add(p.flag, 1u);
        if (p.trace && blockIdx.x == 0) p.trace[i * 8 + 4] = gtimer();
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 32);
  }
}

}  // namespace cmt
