// Recurrent LSTM backward (BPTT) with the W_h slice split across shared
// memory and tensor memory, transposed like lstm_fwd_tm (bf16 path).
//
//   dh_t[b][j] = sum_gc dU_{t+1}[b][gc] W_h[j][gc]          (layers.py:388-392)
//
// is computed as D[j][b] = W_h[j][gc] * dU^T[gc][b]: A = W_h rows of 128 units
// (M = 128, K-major: gate columns contiguous), B = dU rows of a ROWS-row batch
// slice (N = ROWS), K = one quarter of the 4H gate columns.  A cluster of 4
// CTAs (K quarters kq) owns 128 units x ROWS batch rows; its A slice is
// 128 x H bf16 = 256 KB per CTA: 4 k-blocks in smem + 12 in TMEM.  So a CTA
// streams ROWS x H bf16 of dU per step (128 KB at ROWS = 64) where
// lstm_bwd_multi<128> streams 256 KB, with the same 64 CTAs per scan.
//
// Partial sums: TMEM lane quadrant q of every CTA holds the partial of units
// 32q..32q+31, which CTA q of the cluster owns for the cell; each epilogue
// warp pushes its 32 x ROWS/2 block to the owner with st.async (bytes
// complete the owner's mbarrier) into a double-buffered receive area
// [slot][sender][unit][row] that is separate from the TMA ring, so the next
// step's dU stream never waits for the exchange.  The owner adds the four
// partials in sender order (deterministic) and runs the cell backward for its
// 32 units with one batch row and ROWS/8 consecutive units per thread.
// dU k-block pairs (32 units) are published per batch slice with a release
// counter.  Reference semantics: layers.py:366-395 (cell), 472-493 (scan).
#pragma once
#include "lstm_tm.cuh"

namespace cmt {
namespace tmb {
constexpr int THREADS = 384;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-11 epilogue
constexpr int EPI = 8;
constexpr int KS_CL = 4;       // cluster size = K quarters
constexpr int NU = 128;        // units per cluster (MMA M)
constexpr int OU = NU / KS_CL; // units owned (cell) per CTA = 32
constexpr int KBOX = 2;        // k-blocks per stage = 32 units of gate columns = one flag
constexpr int MAX_STAGES = 16;
constexpr size_t SMEM_LIMIT = 227 * 1024;
template <int ROWS>
struct Bwd {
  static constexpr int KBLK = ROWS * 128;                   // [ROWS][64] bf16
  static constexpr int STAGE = KBOX * KBLK;
  static constexpr int XSLOT = KS_CL * OU * ROWS * 4;         // one receive slot [sender][unit][row] fp32
  static constexpr int UPT = ROWS * OU / (EPI * 32);          // units per cell thread
  static constexpr int kt(int H) { return H / 64 < tm::MAX_KT ? H / 64 : tm::MAX_KT; }
  static int ks(int H) { return H / 64 - kt(H); }
  static int stages(int H) {
    long long room = (long long)SMEM_LIMIT - 1024 - 1024 - 2LL * XSLOT - (long long)ks(H) * 16384;
    long long s = room / STAGE;
    return (int)(s > MAX_STAGES ? MAX_STAGES : s);
  }
  static size_t smem(int H) { return 1024 + (size_t)ks(H) * 16384 + 2 * XSLOT + (size_t)stages(H) * STAGE + 1024; }
  static int ctas(int H, int B) { return (H / NU) * KS_CL * ((B + ROWS - 1) / ROWS); }
  static bool ok(int H, int B) {
    return H % NU == 0 && (H / 64) % KBOX == 0 && stages(H) >= 2 && (size_t)stages(H) * STAGE >= 16384 && B >= 1;
  }
};
}  // namespace tmb

template <int ROWS>
__global__ void __launch_bounds__(tmb::THREADS, 1)
    lstm_bwd_tm(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmW0,
                const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmW1,
                const LstmBwdMulti m) {
  using F = tmb::Bwd<ROWS>;
  constexpr int UPT = F::UPT;
  constexpr int CH = ROWS / 2;  // accumulator columns (batch rows) per epilogue warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int ch = (int)blockIdx.x >= m.split ? 1 : 0;
  const LstmBwdP p = ch ? m.c[1] : m.c[0];
  const int bid = ch ? (int)blockIdx.x - m.split : (int)blockIdx.x;
  const void* tmA = ch ? (const void*)&tmA1 : (const void*)&tmA0;
  const void* tmW = ch ? (const void*)&tmW1 : (const void*)&tmW0;

  const int KBL = p.H / 64;  // k-blocks of this CTA's gate-column quarter
  const int KT = F::kt(p.H), KS = KBL - KT;
  uint8_t* sW = smem;                                   // KS x [128 units][64 gc] (K-major)
  float* xbuf = (float*)(smem + (size_t)KS * 16384);    // 2 slots x [4 senders][32 units][ROWS]
  uint8_t* sB = (uint8_t*)xbuf + 2 * F::XSLOT;          // stages x KBOX x [ROWS][64] (K-major)
  uint64_t* full = (uint64_t*)(sB + (size_t)p.stages * F::STAGE);
  uint64_t* empty = full + tmb::MAX_STAGES;
  uint64_t* wfull = empty + tmb::MAX_STAGES;
  uint64_t* sbar = wfull + 1;
  uint64_t* tfull = sbar + 1;
  uint64_t* tempty = tfull + 1;
  uint64_t* xfull = tempty + 1;  // [2]: a slot's three incoming partials have landed
  uint64_t* dfree = xfull + 2;   // [2]: the three partners have consumed what I sent into a slot
  uint32_t* tmem_slot = (uint32_t*)(dfree + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kq = (int)ptx::cluster_rank();
  const int nh = (p.B + ROWS - 1) / ROWS;
  const int cl = bid / tmb::KS_CL;
  const int half = cl % nh;
  const int ug = (cl / nh) * tmb::NU;  // cluster's first unit
  const int r0 = half * ROWS;
  const int kb0g = kq * KBL;           // first global k-block of my gate-column quarter
  const int rounds = p.steps + (p.dh0 ? 1 : 0);
  auto time_of = [&](int pos) { return p.reverse ? p.steps - 1 - pos : pos; };
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(tmA);
    ptx::prefetch_tmap(tmW);
    for (int i = 0; i < p.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(wfull, 1);
    ptx::mbar_init(sbar, 1);
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty, tmb::EPI);
    for (int j = 0; j < 2; ++j) {
      ptx::mbar_init(&xfull[j], 1);                // my expect_tx; partners' st.async bytes complete it
      ptx::mbar_init(&dfree[j], tmb::KS_CL - 1);   // one arrive per partner
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, tm::TMEM_COLS);
  ptx::tc_fence_before();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tA = tmem + tm::D_COLS;

  // ---- W_h slice (units [ug, ug+128), my gate-column quarter): KS k-blocks to
  // smem, KT k-blocks to TMEM through the idle stage ring ----
  const int wrow = p.din + ug;
  if (threadIdx.x == 0 && KS > 0) {
    ptx::mbar_expect_tx(wfull, KS * 16384);
    for (int kb = 0; kb < KS; ++kb) ptx::tma_load_2d(tmW, wfull, sW + kb * 16384, (kb0g + kb) * 64, wrow);
  }
  {
    const int per = (p.stages * F::STAGE) / 16384;
    int round = 0;
    for (int k0 = 0; k0 < KT; k0 += per, ++round) {
      const int nk = KT - k0 < per ? KT - k0 : per;
      if (threadIdx.x == 0) {
        ptx::mbar_expect_tx(sbar, nk * 16384);
        for (int i = 0; i < nk; ++i) ptx::tma_load_2d(tmW, sbar, sB + i * 16384, (kb0g + KS + k0 + i) * 64, wrow);
      }
      if (warp >= 4 && warp < 8) {
        ptx::mbar_wait(sbar, round & 1);
        const int mrow = (warp & 3) * 32 + lane;  // unit row = TMEM lane
        for (int i = 0; i < nk; ++i) {
          const uint8_t* rowp = sB + i * 16384 + mrow * 128;
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < 32; ++c)  // bf16 pair (2c, 2c+1) sits in 16-byte chunk c/4 ^ (row & 7)
            r[c] = *(const uint32_t*)(rowp + ((((c >> 2) ^ (mrow & 7)) << 4) | ((c & 3) << 2)));
          tm::tmem_st32(tA + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((k0 + i) * 32), r);
        }
        tm::tmem_wait_st();
      }
      __syncthreads();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();

  if (warp == 0) {
    // ===== producer: dU rows of round i-1 for my batch slice and gate-column
    // quarter; stage s (32 units) is ready once its owner published round i-1 =====
    int stage = 0;
    uint32_t phase = 0;
    const int nst = KBL / tmb::KBOX;
    const int fb0 = kb0g / tmb::KBOX;  // first 32-unit block of my quarter
    for (int i = 1; i < rounds; ++i) {
      const int arow = time_of(p.steps - i) * p.B + r0;
      const unsigned target = (unsigned)i;
      int issued = 0;
      while (issued < nst) {
        const bool ok = lane >= nst || ptx::ld_acquire(p.flag + (fb0 + lane) * nh + half) >= target;
        const unsigned ready = __ballot_sync(0xffffffffu, ok);
        __syncwarp();
        if (lane == 0) {
          ptx::fence_proxy_async_global();
          while (issued < nst && ((ready >> issued) & 1u)) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            if (p.trace && bid == 0 && (issued == 0 || issued == nst - 1)) p.trace[i * 8 + (issued ? 6 : 5)] = gtimer();
            ptx::tma_load_3d(tmA, &full[stage], sB + stage * F::STAGE, 0, arow, kb0g + issued * tmb::KBOX);
            ptx::mbar_expect_tx(&full[stage], F::STAGE);
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
            ++issued;
          }
        }
        issued = __shfl_sync(0xffffffffu, issued, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, ROWS, 0, 0);
      if (KS > 0) ptx::mbar_wait(wfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t wbase = ptx::smem_u32(sW);
      for (int i = 1; i < rounds; ++i) {
        ptx::mbar_wait(tempty, ((i - 1) & 1) ^ 1);
        ptx::tc_fence_after();
        for (int kb0 = 0; kb0 < KBL; kb0 += tmb::KBOX) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (p.trace && bid == 0 && kb0 + tmb::KBOX >= KBL) p.trace[i * 8 + 7] = gtimer();
          const uint32_t b0 = ptx::smem_u32(sB + stage * F::STAGE);
#pragma unroll
          for (int j = 0; j < tmb::KBOX; ++j) {
            const int kb = kb0 + j;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t bd = ptx::smem_desc_sw128(b0 + j * F::KBLK + kk * 32, 16, 1024);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              if (kb < KS) {
                const uint64_t ad = ptx::smem_desc_sw128(wbase + kb * 16384 + kk * 32, 16, 1024);
                ptx::umma_bf16(tmem, ad, bd, idesc, acc);
              } else {
                tm::umma_bf16_ts(tmem, tA + (uint32_t)((kb - KS) * 32 + kk * 8), bd, idesc, acc);
              }
            }
          }
          ptx::umma_commit(&empty[stage]);
          if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(tfull);
      }
    }
  } else if (warp >= 4) {
    const int e = warp - 4;
    // exchange role: TMEM lane quadrant q (units ug + 32q + lane), columns [hc*CH, hc*CH + CH)
    const int q = e & 3, hc = e >> 2;
    // cell role: batch row cb, units uo*UPT .. +UPT of my 32 owned units
    constexpr int RW = ROWS / 32;  // warps per unit group in the cell role
    const int cb = (e % RW) * 32 + lane;
    const int uo = e / RW;
    const bool valid = r0 + cb < p.B;
    const long long gb = r0 + cb;
    const long long H = p.H;
    const int u0 = ug + kq * tmb::OU + uo * UPT;  // my cell units
    // remote addresses: receive area of CTA q (slot base; sender = my kq), its xfull, partners' dfree
    const uint32_t xb_local = ptx::smem_u32(xbuf);
    uint32_t rdf[tmb::KS_CL];
#pragma unroll
    for (int pr_ = 0; pr_ < tmb::KS_CL; ++pr_) rdf[pr_] = ptx::mapa(ptx::smem_u32(dfree), pr_);
    const uint32_t rx_base = ptx::mapa(xb_local, q) + (uint32_t)(((kq * tmb::OU + lane) * ROWS + hc * CH) * 4);
    const uint32_t rxf_base = ptx::mapa(ptx::smem_u32(xfull), q);
    float dhc[UPT], dc[UPT];
#pragma unroll
    for (int u = 0; u < UPT; ++u) {
      dhc[u] = (valid && p.dh_final) ? p.dh_final[gb * H + u0 + u] : 0.f;
      dc[u] = (valid && p.dc_final) ? p.dc_final[gb * H + u0 + u] : 0.f;
    }
    for (int i = 0; i < rounds; ++i) {
      const bool cell = i < p.steps;
      const int t = cell ? time_of(p.steps - 1 - i) : 0;
      const long long row = (long long)t * p.B + gb;
      // prefetch the cell operands (independent of the recurrent sum)
      float dyv[UPT], tcv[UPT], cpv[UPT];
      float4 a4[UPT];
      float mk = 1.f;
      if (valid && cell) {
#pragma unroll
        for (int k = 0; k < UPT / 4; ++k) {
          const float4 d = __ldg((const float4*)(p.dy + row * H + u0) + k);
          const float4 tcx = __ldg((const float4*)(p.tcache + row * H + u0) + k);
          const float4 cp = __ldg((const float4*)(p.cprev + row * H + u0) + k);
          dyv[4 * k] = d.x; dyv[4 * k + 1] = d.y; dyv[4 * k + 2] = d.z; dyv[4 * k + 3] = d.w;
          tcv[4 * k] = tcx.x; tcv[4 * k + 1] = tcx.y; tcv[4 * k + 2] = tcx.z; tcv[4 * k + 3] = tcx.w;
          cpv[4 * k] = cp.x; cpv[4 * k + 1] = cp.y; cpv[4 * k + 2] = cp.z; cpv[4 * k + 3] = cp.w;
        }
#pragma unroll
        for (int u = 0; u < UPT; ++u) a4[u] = __ldg((const float4*)(p.acts + row * 4 * H + 4 * u0) + u);
        if (p.mask) mk = __ldg(p.mask + row);
      }
      float acc[UPT];
#pragma unroll
      for (int u = 0; u < UPT; ++u) acc[u] = 0.f;
      if (i > 0) {
        const int slot = i & 1;
        const uint32_t use = (uint32_t)((i - 1) >> 1) & 1u;  // parity of this slot's use
        ptx::mbar_wait(tfull, (i - 1) & 1);
        ptx::tc_fence_after();
        if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[i * 8 + 1] = gtimer();
        float v[CH];
#pragma unroll
        for (int c0 = 0; c0 < CH; c0 += 16)
          ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + hc * CH + c0, v + c0);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tempty);
        if (threadIdx.x == 128) ptx::mbar_expect_tx(&xfull[slot], (tmb::KS_CL - 1) * tmb::OU * ROWS * 4);
        if (q == kq) {  // my own units: straight into my receive slot
          float* dst = xbuf + slot * (F::XSLOT / 4) + (kq * tmb::OU + lane) * ROWS + hc * CH;
#pragma unroll
          for (int c = 0; c < CH; c += 4) *(float4*)(dst + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
        } else {
          // the owner must have consumed what I sent into this slot two rounds ago
          ptx::mbar_wait_cluster(&dfree[slot], use ^ 1);
          const uint32_t dst = rx_base + (uint32_t)(slot * F::XSLOT);
          const uint32_t bar = rxf_base + (uint32_t)(slot * 8);
#pragma unroll
          for (int c = 0; c < CH; c += 4) ptx::st_async_v4(dst + c * 4, v[c], v[c + 1], v[c + 2], v[c + 3], bar);
        }
        ptx::named_bar_sync(1, 32 * tmb::EPI);  // my own block is in the slot
        ptx::mbar_wait_cluster(&xfull[slot], use);
        if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[i * 8 + 2] = gtimer();
        const float* xs = xbuf + slot * (F::XSLOT / 4);
#pragma unroll
        for (int s = 0; s < tmb::KS_CL; ++s)  // fixed sender order: deterministic sum
#pragma unroll
          for (int u = 0; u < UPT; ++u) acc[u] += xs[(s * tmb::OU + uo * UPT + u) * ROWS + cb];
      }
      if (valid) {
        if (cell) {
          __align__(16) bf16 du[4 * UPT];
#pragma unroll
          for (int u = 0; u < UPT; ++u) {
            const float dh = acc[u] + dhc[u] + dyv[u];
            float dhn = dh, dcn = dc[u], dhcar = 0.f, dccar = 0.f;
            if (p.mask) {
              dhn = mk * dh; dcn = mk * dc[u];
              dhcar = (1.f - mk) * dh; dccar = (1.f - mk) * dc[u];
            }
            const float4 a = a4[u];  // i f g o
            const float tc = tcv[u];
            const float dct = dhn * a.w * (1.f - tc * tc) + dcn;
            du[4 * u + 0] = __float2bfloat16_rn(dct * a.z * (a.x * (1.f - a.x)));
            du[4 * u + 1] = __float2bfloat16_rn(dct * cpv[u] * (a.y * (1.f - a.y)));
            du[4 * u + 2] = __float2bfloat16_rn(dct * a.x * (1.f - a.z * a.z));
            du[4 * u + 3] = __float2bfloat16_rn(dhn * tc * (a.w * (1.f - a.w)));
            dc[u] = dct * a.y + dccar;
            dhc[u] = dhcar;
          }
          uint4* dur = (uint4*)(p.dU + row * 4 * H + 4 * u0);
#pragma unroll
          for (int k = 0; k < UPT / 2; ++k) dur[k] = ((uint4*)du)[k];
        } else {
#pragma unroll
          for (int u = 0; u < UPT; ++u) {
            p.dh0[gb * H + u0 + u] = acc[u] + dhc[u];
            p.dc0[gb * H + u0 + u] = dc[u];
          }
        }
      }
      if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[i * 8 + 3] = gtimer();
      ptx::named_bar_sync(1, 32 * tmb::EPI);
      if (threadIdx.x == 128) {
        // my 32 units of dU (one k-block pair) for this batch slice
        ptx::red_release_add(p.flag + ((ug + kq * tmb::OU) >> 5) * nh + half, 1u);
        if (p.trace && bid == 0) p.trace[i * 8 + 4] = gtimer();
        if (i > 0) {  // the partners may reuse this round's slot of my receive area
#pragma unroll
          for (int pr_ = 0; pr_ < tmb::KS_CL; ++pr_)
            if (pr_ != kq) ptx::mbar_arrive_remote(rdf[pr_] + (uint32_t)((i & 1) * 8));
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();  // no CTA leaves while a partner may still write into its receive area
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, tm::TMEM_COLS);
  }
}

}  // namespace cmt
