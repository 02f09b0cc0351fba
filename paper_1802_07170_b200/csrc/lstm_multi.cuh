// Multi-chain persistent recurrent LSTM forward (bf16 production path).
//
// Same per-CTA contract as lstm_fwd_persistent (W_h slice resident in smem,
// h_{t-1} streamed by TMA into a stage ring, tcgen05.mma into TMEM, fused cell
// epilogue with c/h in registers, grid step counter instead of launches), but
// one cooperative launch runs up to two INDEPENDENT scans side by side on
// disjoint CTA ranges.  The encoder/decoder layer graph has two independent
// scans at every level (enc.l1 fwd || bwd, enc.l(k+1) || dec.lk), so the
// forward's critical path shrinks from 2L+1 scans to L+1.
//
// ROWS = batch rows per CTA.  ROWS = 128 (whole batch, 64 CTAs per chain at
// H=1024) is the paired configuration: each CTA streams the full h_{t-1}
// (B x H bf16) per step and every accumulator row is useful.  ROWS = 64 splits
// the batch over two CTAs (128 CTAs, the single-chain configuration).
// Reference semantics: layers.py:344-363 (cell), layers.py:440-470 (scan).
#pragma once
#include "lstm_common.cuh"

namespace cmt {
namespace mc {
constexpr int THREADS = 256;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4.. cell epilogue (ROWS/32 warps)
constexpr int MAX_STAGES = 8;
constexpr int STAGE_BYTES = 32 * 1024;
constexpr int FWD_NG = 64;  // gate columns (16 units) per CTA
constexpr size_t SMEM_LIMIT = 227 * 1024;
template <int ROWS>
struct Fwd {
  static constexpr int KBLK = ROWS * 128;            // [ROWS rows][64] bf16 k-block tile
  static constexpr int KBOX = STAGE_BYTES / KBLK;    // k-blocks per (3-D) TMA = one stage
  static constexpr int PAD = ROWS < 128 ? KBLK : 0;  // UMMA M=128 reads 128 rows past the last tile
  static int stages(int H) {
    long long room = (long long)SMEM_LIMIT - 1024 - 256 - PAD - (long long)H * 128;
    long long s = room / STAGE_BYTES;
    return (int)(s > MAX_STAGES ? MAX_STAGES : s);
  }
  static size_t smem(int H) { return 1024 + (size_t)H * 128 + (size_t)stages(H) * STAGE_BYTES + PAD + 256; }
  static int ctas(int H, int B) { return (4 * H / FWD_NG) * ((B + ROWS - 1) / ROWS); }
};
}  // namespace mc

struct LstmFwdMulti {
  LstmFwdP c[2];
  int split;  // CTAs [0, split) run chain 0, [split, grid) chain 1
};

template <int ROWS>
__global__ void __launch_bounds__(mc::THREADS, 1)
    lstm_fwd_multi(const __grid_constant__ CUtensorMap tmH0, const __grid_constant__ CUtensorMap tmW0,
                   const __grid_constant__ CUtensorMap tmH1, const __grid_constant__ CUtensorMap tmW1,
                   const LstmFwdMulti m) {
  using F = mc::Fwd<ROWS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int ch = (int)blockIdx.x >= m.split ? 1 : 0;
  const LstmFwdP p = ch ? m.c[1] : m.c[0];
  const int bid = ch ? (int)blockIdx.x - m.split : (int)blockIdx.x;
  const int G = ch ? (int)gridDim.x - m.split : m.split;
  const void* tmH = ch ? (const void*)&tmH1 : (const void*)&tmH0;
  const void* tmW = ch ? (const void*)&tmW1 : (const void*)&tmW0;

  const int KB = p.H / 64;
  uint8_t* sW = smem;                      // KB x [64 K rows][64 N] (MN-major atoms)
  uint8_t* sA = smem + (size_t)KB * 8192;  // stages x KBOX x [ROWS][64] (K-major) + pad
  uint64_t* full = (uint64_t*)(sA + p.stages * mc::STAGE_BYTES + F::PAD);
  uint64_t* empty = full + mc::MAX_STAGES;
  uint64_t* wfull = empty + mc::MAX_STAGES;
  uint64_t* tfull = wfull + 1;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);
  constexpr int EPI_W = ROWS / 32;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nh = (p.B + ROWS - 1) / ROWS;
  const int half = bid % nh;
  const int n0 = (bid / nh) * mc::FWD_NG;
  const int u0 = n0 >> 2;
  const int r0 = half * ROWS;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(tmH);
    ptx::prefetch_tmap(tmW);
    for (int i = 0; i < p.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(wfull, 1);
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty, EPI_W);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 64);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===== producer (whole warp): h_{t-1} k-block kb is ready once its 4
    // producer CTAs (units [64kb, 64kb+64), this batch half) have bumped
    // flag[kb * nh + half] for the previous step; lanes poll the flags in
    // parallel and lane 0 streams every stage whose k-blocks are ready, so
    // the first k-blocks load while the slowest producers are still finishing.
    if (lane == 0) {
      ptx::mbar_expect_tx(wfull, KB * 8192);
      for (int kb = 0; kb < KB; ++kb) ptx::tma_load_2d(tmW, wfull, sW + kb * 8192, n0, p.din + kb * 64);
    }
    int stage = 0;
    uint32_t phase = 0;
    const int nst = KB / F::KBOX;
    for (int s = 0; s < p.steps; ++s) {
      const int t = p.reverse ? p.steps - 1 - s : s;
      if (p.trace && bid == 0 && lane == 0) p.trace[s * 8 + 0] = gtimer();
      const int hrow = p.hrow0 + t * p.B + r0;
      const unsigned target = 4u * (unsigned)s;
      int issued = 0;
      SpinGuard guard;
      while (issued < nst) {
        unsigned ready = 0xffffffffu;
        if (s > 0) {
          const bool ok = lane >= KB || ptx::ld_acquire(p.flag + lane * nh + half) >= target;
          ready = __ballot_sync(0xffffffffu, ok);
          __syncwarp();
          if (ready != 0xffffffffu && __shfl_sync(0xffffffffu, lane == 0 ? (int)guard.expired(p.status) : 0, 0))
            ready = 0xffffffffu;  // wait budget exceeded: the step is reported failed  // order the lanes' acquire loads before lane 0's TMA issue
        }
        if (lane == 0) {
          if (s > 0) ptx::fence_proxy_async_global();
          while (issued < nst) {
            const unsigned need = ((1u << F::KBOX) - 1u) << (issued * F::KBOX);
            if ((ready & need) != need) break;
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            if (p.trace && bid == 0 && (issued == 0 || issued == nst - 1)) p.trace[s * 8 + (issued ? 5 : 4)] = gtimer();
            ptx::tma_load_3d(tmH, &full[stage], sA + stage * mc::STAGE_BYTES, 0, hrow, issued * F::KBOX);
            ptx::mbar_expect_tx(&full[stage], mc::STAGE_BYTES);
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
            ++issued;
          }
        }
        issued = __shfl_sync(0xffffffffu, issued, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16(128, mc::FWD_NG, 0, 1);
      ptx::mbar_wait(wfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t wbase = ptx::smem_u32(sW);
      for (int s = 0; s < p.steps; ++s) {
        ptx::mbar_wait(tempty, (s & 1) ^ 1);
        ptx::tc_fence_after();
        for (int kb0 = 0; kb0 < KB; kb0 += F::KBOX) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (p.trace && bid == 0 && (kb0 == 0 || kb0 + F::KBOX >= KB)) p.trace[s * 8 + (kb0 ? 7 : 6)] = gtimer();
          const uint32_t a0 = ptx::smem_u32(sA + stage * mc::STAGE_BYTES);
#pragma unroll
          for (int j = 0; j < F::KBOX; ++j) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint64_t ad = ptx::smem_desc_sw128(a0 + j * F::KBLK + kk * 32, 16, 1024);
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
  } else if (warp >= 4 && warp < 4 + EPI_W) {
    const int q = warp & 3;
    const int b = r0 + q * 32 + lane;
    const bool valid = b < p.B;
    const long long H = p.H;
    float c[16], h[16];
    {
      const int t0 = p.reverse ? p.steps - 1 : 0;
      const long long rr = (long long)t0 * p.B + b;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        c[u] = valid ? p.cprev[rr * H + u0 + u] : 0.f;
        h[u] = valid ? __bfloat162float(p.hprev[rr * H + u0 + u]) : 0.f;
      }
    }
    for (int s = 0; s < p.steps; ++s) {
      const int t = p.reverse ? p.steps - 1 - s : s;
      const long long row = (long long)t * p.B + b;
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
      if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[s * 8 + 1] = gtimer();
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
      if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[s * 8 + 2] = gtimer();
      // publish h_t (the only value other CTAs need), then write the BPTT caches
      ptx::named_bar_sync(1, ROWS);
      if (threadIdx.x == 128) {
        ptx::red_release_add(p.flag + (u0 >> 6) * nh + half, 1u);
        if (p.trace && bid == 0) p.trace[s * 8 + 3] = gtimer();
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

// ---------------------------------------------------------------------------
// Multi-chain cluster K-split recurrent backward (BPTT) kernel.
//
// dh_t[b][j] = sum_gc dU_{t+1}[b][gc] W_h[j][gc]: a cluster of 4 CTAs owns 64
// units; CTA rank kq contracts the gate columns [kq*H, (kq+1)*H) of dU_{t+1}
// for all 64 units (M = B <= 128 rows, N = 64, K = H) with its W_h slice
// resident in smem, then the four partial sums are combined through
// distributed shared memory: once a CTA's MMA is done its (idle) TMA stage
// ring can receive, and each CTA pushes every partner the slice of partials
// for the partner's 16 units with st.async (bytes complete the partner's
// mbarrier, so no cluster fence is paid per step).  8 epilogue warps run the cell backward for
// 16 units x 128 rows.  Two independent scans can share one cooperative
// launch (the backward layer graph pairs dec.lk with enc.l(k+1), and
// enc.l1 bwd with enc.l1 fwd).  Reference: layers.py:366-395, 472-493.
// ---------------------------------------------------------------------------
namespace mc {
constexpr int BWD_NU = 64;        // units per cluster
constexpr int BWD_UPT = 8;        // units per epilogue thread
constexpr int BWD_KBOX = 2;       // k-blocks per TMA / stage
// ROWS = batch rows per CTA: 128 (paired scans) or 64 (one scan split over two
// batch halves, 128 CTAs; the M=128 MMA reads a padding tile past the stage).
// KS = cluster size = K slices of the 4H gate columns (4 or 8): each CTA holds
// a (4H/KS) x 64-unit W_h slice and streams 1/KS of dU per step; a larger KS
// halves both, leaving room for twice the TMA stages in flight, at the price
// of more (smaller) partial sums in the exchange.
template <int ROWS, int KS>
struct Bwd {
  static constexpr int UPC = BWD_NU / KS;          // units per CTA (16 or 8)
  static constexpr int NG = UPC / BWD_UPT;         // 8-unit groups per CTA (2 or 1)
  static constexpr int EPI_WARPS = 4 * NG;       // warp w: TMEM lane quarter w & 3, unit group (w - 4) >> 2
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;  // w0 TMA, w1 MMA, w2 TMEM, w3 idle, epilogue
  static constexpr int KBLK = ROWS * 128;  // [ROWS rows][64] bf16
  static constexpr int STAGE = BWD_KBOX * KBLK;
  static constexpr int PAD = ROWS < 128 ? KBLK : 0;
  static constexpr int PROD = 16 / UPC;            // CTAs producing one 64-column k-block of dU
  static size_t w_bytes(int H) { return (size_t)(4 * H / 64 / KS) * BWD_NU * 128; }
  static int stages(int H) {
    long long room = (long long)SMEM_LIMIT - 1024 - 512 - PAD - (long long)w_bytes(H);
    long long s = room / STAGE;
    return (int)(s > MAX_STAGES ? MAX_STAGES : s);
  }
  static size_t smem(int H) { return 1024 + w_bytes(H) + (size_t)stages(H) * STAGE + PAD + 512; }
  static int ctas(int H, int B) { return (H / BWD_NU) * KS * ((B + ROWS - 1) / ROWS); }
  static size_t xbuf_bytes() { return (size_t)KS * NG * ROWS * 32; }
};
}  // namespace mc

struct LstmBwdMulti {
  LstmBwdP c[2];
  int split;  // multiple of the cluster size
};

template <int ROWS, int KS>
__global__ void __launch_bounds__(mc::Bwd<ROWS, KS>::THREADS, 1)
    lstm_bwd_multi(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmW0,
                   const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmW1,
                   const LstmBwdMulti m) {
  using F = mc::Bwd<ROWS, KS>;
  constexpr int UPC = F::UPC, NG = F::NG, EPI_WARPS = F::EPI_WARPS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int ch = (int)blockIdx.x >= m.split ? 1 : 0;
  const LstmBwdP p = ch ? m.c[1] : m.c[0];
  const int bid = ch ? (int)blockIdx.x - m.split : (int)blockIdx.x;
  const int G = ch ? (int)gridDim.x - m.split : m.split;
  const void* tmA = ch ? (const void*)&tmA1 : (const void*)&tmA0;
  const void* tmW = ch ? (const void*)&tmW1 : (const void*)&tmW0;

  const int KBL = 4 * p.H / 64 / KS;  // k-blocks of this CTA's gate-column slice
  uint8_t* sW = smem;                                    // KBL x [64 units][64] (K-major)
  uint8_t* sA = smem + (size_t)KBL * (mc::BWD_NU * 128);  // stage ring; also the parked partials
  uint64_t* full = (uint64_t*)(sA + (size_t)p.stages * F::STAGE + F::PAD);
  uint64_t* empty = full + mc::MAX_STAGES;
  uint64_t* wfull = empty + mc::MAX_STAGES;
  uint64_t* tfull = wfull + 1;
  uint64_t* tempty = tfull + 1;
  uint64_t* rfree = tempty + 1;  // the three partners' MMAs are done: their rings may receive partials
  uint64_t* xfull = rfree + 1;   // all partials for my units have landed in my ring
  uint64_t* xdone = xfull + 1;   // my epilogue has read this round's partials: the ring may refill
  uint32_t* tmem_slot = (uint32_t*)(xdone + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kq = (int)ptx::cluster_rank();
  const int nh = (p.B + ROWS - 1) / ROWS;
  const int half = (bid / KS) % nh;                  // batch half of this cluster
  const int ug = (bid / KS / nh) * mc::BWD_NU;       // cluster's first unit
  const int r0 = half * ROWS;
  const int kb_base = kq * KBL;
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
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty, EPI_WARPS);
    ptx::mbar_init(rfree, KS - 1);
    ptx::mbar_init(xfull, 1);  // my expect_tx; the partners' st.async bytes complete it
    ptx::mbar_init(xdone, EPI_WARPS);  // the epilogue warps
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 64);
  ptx::tc_fence_before();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===== producer (whole warp): k-block kb of dU (gate columns [64kb, 64kb+64)
    // = 16 units) is written by exactly one CTA, which bumps flag[kb] once per
    // round; lanes poll this CTA's KBL flags in parallel and lane 0 streams
    // every stage whose k-blocks are ready (no grid-wide step barrier).
    if (lane == 0) {
      ptx::mbar_expect_tx(wfull, KBL * mc::BWD_NU * 128);
      for (int kb = 0; kb < KBL; ++kb)
        ptx::tma_load_2d(tmW, wfull, sW + kb * (mc::BWD_NU * 128), (kb_base + kb) * 64, p.din + ug);
    }
    int stage = 0;
    uint32_t phase = 0;
    const int nst = KBL / mc::BWD_KBOX;
    for (int i = 1; i < rounds; ++i) {
      // the ring doubles as the receive buffer of round i-1's partial sums: with
      // per-k-block flags this round's k-blocks can be ready before this CTA has
      // read them, so wait until its epilogue is done with the partials
      if (i >= 2) ptx::mbar_wait(xdone, (i - 2) & 1);
      if (p.trace && bid == 0 && lane == 0) p.trace[i * 8 + 0] = gtimer();
      const int arow = time_of(p.steps - i) * p.B + r0;
      const unsigned target = (unsigned)(i * F::PROD);
      int issued = 0;
      SpinGuard guard;
      while (issued < nst) {
        const bool ok = lane >= KBL || ptx::ld_acquire(p.flag + (kb_base + lane) * nh + half) >= target;
        unsigned ready = __ballot_sync(0xffffffffu, ok);
        __syncwarp();
        if (ready != 0xffffffffu && __shfl_sync(0xffffffffu, lane == 0 ? (int)guard.expired(p.status) : 0, 0))
          ready = 0xffffffffu;  // wait budget exceeded: the step is reported failed
        if (lane == 0) {
          ptx::fence_proxy_async_global();
          ptx::fence_proxy_async_shared();
          while (issued < nst) {
            const unsigned need = ((1u << mc::BWD_KBOX) - 1u) << (issued * mc::BWD_KBOX);
            if ((ready & need) != need) break;
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            if (p.trace && bid == 0 && (issued == 0 || issued == nst - 1)) p.trace[i * 8 + (issued ? 6 : 5)] = gtimer();
            ptx::tma_load_3d(tmA, &full[stage], sA + stage * F::STAGE, 0, arow, kb_base + issued * mc::BWD_KBOX);
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
      const uint32_t idesc = ptx::idesc_bf16(128, mc::BWD_NU, 0, 0);
      ptx::mbar_wait(wfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t wbase = ptx::smem_u32(sW);
      for (int i = 1; i < rounds; ++i) {
        ptx::mbar_wait(tempty, ((i - 1) & 1) ^ 1);
        ptx::tc_fence_after();
        for (int kb0 = 0; kb0 < KBL; kb0 += mc::BWD_KBOX) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (p.trace && bid == 0 && kb0 + mc::BWD_KBOX >= KBL) p.trace[i * 8 + 7] = gtimer();
          const uint32_t a0 = ptx::smem_u32(sA + stage * F::STAGE);
#pragma unroll
          for (int j = 0; j < mc::BWD_KBOX; ++j) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              uint64_t ad = ptx::smem_desc_sw128(a0 + j * F::KBLK + kk * 32, 16, 1024);
              uint64_t bd = ptx::smem_desc_sw128(wbase + (kb0 + j) * (mc::BWD_NU * 128) + kk * 32, 16, 1024);
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
    const int uh = (warp - 4) >> 2;  // 8-unit group of this CTA's units
    const int b = q * 32 + lane;               // row within this CTA's batch slice
    const bool inrow = b < ROWS;
    const bool valid = inrow && r0 + b < p.B;
    const long long gb = r0 + b;                // batch column
    const long long H = p.H;
    const int u0 = ug + kq * UPC + uh * 8;  // my 8 units
    // partials parked in the receiver's stage ring: xbuf[sender][uh][row][8] floats
    const uint32_t xslot = ptx::smem_u32(sA) + (uint32_t)((kq * NG + uh) * ROWS + (inrow ? b : 0)) * 32;
    uint32_t rx[KS], rxf[KS], rrf[KS];
#pragma unroll
    for (int pr_ = 0; pr_ < KS; ++pr_) {
      rx[pr_] = ptx::mapa(xslot, pr_);
      rxf[pr_] = ptx::mapa(ptx::smem_u32(xfull), pr_);
      rrf[pr_] = ptx::mapa(ptx::smem_u32(rfree), pr_);
    }
    float dhc[mc::BWD_UPT], dc[mc::BWD_UPT];
#pragma unroll
    for (int u = 0; u < mc::BWD_UPT; ++u) {
      dhc[u] = (valid && p.dh_final) ? p.dh_final[gb * H + u0 + u] : 0.f;
      dc[u] = (valid && p.dc_final) ? p.dc_final[gb * H + u0 + u] : 0.f;
    }
    for (int i = 0; i < rounds; ++i) {
      const bool cell = i < p.steps;
      const int t = cell ? time_of(p.steps - 1 - i) : 0;
      const long long row = (long long)t * p.B + gb;
      float4 dy4[2], tc4[2], cp4[2], a4[mc::BWD_UPT];
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
        for (int u = 0; u < mc::BWD_UPT; ++u) a4[u] = __ldg(ar + u);
        if (p.mask) mk = __ldg(p.mask + row);
      }
      float acc[mc::BWD_UPT];
      if (i > 0) {
        ptx::mbar_wait(tfull, (i - 1) & 1);
        ptx::tc_fence_after();
        if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[i * 8 + 1] = gtimer();
        if (p.trace && bid < 8 && threadIdx.x == 128) p.trace[1024 + i * 8 + bid] = gtimer();
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
        float v[KS][mc::BWD_UPT];
#pragma unroll
        for (int pr_ = 0; pr_ < KS; ++pr_) ptx::tmem_ld8(tl + pr_ * UPC + uh * 8, v[pr_]);
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tempty);
        // my MMA is done: my ring may now receive the partners' partials
        if (threadIdx.x == 128) {
          ptx::mbar_expect_tx(xfull, (KS - 1) * NG * ROWS * 32);
#pragma unroll
          for (int pr_ = 0; pr_ < KS; ++pr_)
            if (pr_ != kq) ptx::mbar_arrive_remote_relaxed(rrf[pr_]);
        }
#pragma unroll
        for (int pr_ = 0; pr_ < KS; ++pr_)
          if (pr_ == kq) {
#pragma unroll
            for (int u = 0; u < mc::BWD_UPT; ++u) acc[u] = v[pr_][u];
          }
        // push each partner its 8 columns (async remote stores completing its xfull)
        ptx::mbar_wait_cluster(rfree, (i - 1) & 1);
#pragma unroll
        for (int pr_ = 0; pr_ < KS; ++pr_) {
          if (pr_ == kq || !inrow) continue;
          ptx::st_async_v4(rx[pr_], v[pr_][0], v[pr_][1], v[pr_][2], v[pr_][3], rxf[pr_]);
          ptx::st_async_v4(rx[pr_] + 16, v[pr_][4], v[pr_][5], v[pr_][6], v[pr_][7], rxf[pr_]);
        }
        ptx::mbar_wait_cluster(xfull, (i - 1) & 1);
#pragma unroll
        for (int pr_ = 0; pr_ < KS; ++pr_) {
          if (pr_ == kq || !inrow) continue;
          const float4* xr = (const float4*)(sA + ((pr_ * NG + uh) * ROWS + b) * 32);
          const float4 z0 = xr[0], z1 = xr[1];
          acc[0] += z0.x; acc[1] += z0.y; acc[2] += z0.z; acc[3] += z0.w;
          acc[4] += z1.x; acc[5] += z1.y; acc[6] += z1.z; acc[7] += z1.w;
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(xdone);  // partials consumed: the producer may refill the ring
        if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[i * 8 + 2] = gtimer();
      } else {
#pragma unroll
        for (int u = 0; u < mc::BWD_UPT; ++u) acc[u] = 0.f;
      }
      if (valid) {
        if (cell) {
          __align__(16) bf16 du[4 * mc::BWD_UPT];
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
          for (int k = 0; k < 4; ++k) dur[k] = ((uint4*)du)[k];
        } else {
#pragma unroll
          for (int u = 0; u < mc::BWD_UPT; ++u) {
            p.dh0[gb * H + u0 + u] = acc[u] + dhc[u];
            p.dc0[gb * H + u0 + u] = dc[u];
          }
        }
      }
      if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[i * 8 + 3] = gtimer();
      ptx::named_bar_sync(1, 32 * EPI_WARPS);
      if (threadIdx.x == 128) {
        // my units' gate columns 4*(ug + UPC kq) .. lie in k-block (ug + UPC kq) / 16 of
        // this batch half (shared by PROD = 16 / UPC CTAs)
        ptx::red_release_add(p.flag + ((ug + kq * UPC) >> 4) * nh + half, 1u);
        if (p.trace && bid == 0) p.trace[i * 8 + 4] = gtimer();
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();  // no CTA leaves while a partner may still write into its ring
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 64);
  }
}

}  // namespace cmt
