// Recurrent LSTM forward with the W_h slice split across shared memory AND
// tensor memory (bf16 production path).
//
// The per-step cost of the persistent scans is dominated by streaming
// h_{t-1} into every CTA (B x H bf16 per step per CTA: 256 KB at B=128,
// H=1024).  Halving the streamed rows needs twice the resident weights per
// CTA, which shared memory alone cannot hold (128 gate columns x H = 256 KB).
// tcgen05.mma accepts its A operand from TMEM, so the problem is transposed:
//
//   D[gc][b] = sum_k W_h[k][n0+gc] * h_{t-1}[r0+b][k]     M = 128 gate columns,
//                                                          N = ROWS batch rows, K = H
//
// A = W_h slice (gate columns x K): the first KS k-blocks stay in smem
// (MN-major, 128B-swizzled TMA atoms), the last KT k-blocks live in TMEM
// (lane = gate column, bf16 pairs along columns), both loaded once per scan.
// B = h_{t-1} rows of this CTA's batch slice (K-major tiles by 3-D TMA), so a
// CTA streams ROWS x H bf16 per step: 128 KB at ROWS=64, half the 128-row
// kernel's stream, with the same 64 CTAs per scan (paired scans still fit).
//
// Epilogue: 4 warps, thread = gate column (TMEM lane).  Gate pre-activations
// (+ hoisted input projection) are activated per thread, transposed through a
// small smem tile so that warp q / lane j owns unit j for batch rows q + 4i,
// and the cell update runs with c/h carried in registers.  h_t is published
// per k-block with a release counter (2 producer CTAs per 64-unit k-block and
// batch slice) exactly like lstm_fwd_multi.  Reference semantics:
// layers.py:344-363 (cell), layers.py:440-470 (masked scan).
#pragma once
#include "lstm_multi.cuh"

namespace cmt {
namespace tm {
constexpr int THREADS = 384;   // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-11 epilogue
constexpr int EPI = 8;         // epilogue warps: 2 per TMEM lane quadrant
constexpr int NG = 128;        // gate columns per CTA (32 units)
constexpr int NU = NG / 4;
constexpr int MAX_STAGES = 8;
constexpr int TMEM_COLS = 512;
constexpr int D_COLS = 128;    // accumulator columns reserved (N = ROWS <= 128)
#ifndef CMT_TM_MAX_KT
#define CMT_TM_MAX_KT ((TMEM_COLS - D_COLS) / 32)
#endif
constexpr int MAX_KT = CMT_TM_MAX_KT;  // k-blocks of W_h held in TMEM (the rest in smem)
constexpr size_t SMEM_LIMIT = 227 * 1024;
template <int ROWS>
struct Fwd {
  static constexpr int KBLK = ROWS * 128;  // [ROWS rows][64] bf16 k-block tile
  static constexpr int KBOX = ROWS >= 64 ? 4 : 4;
  static constexpr int STAGE = KBOX * KBLK;
  static constexpr int TBYTES = ROWS * NG * 4;  // transpose tile [ROWS][NG] fp32
  static CMT_HD int kt(int H) { return H / 64 < MAX_KT ? H / 64 : MAX_KT; }
  static int ks(int H) { return H / 64 - kt(H); }
  static int stages(int H) {
    long long room = (long long)SMEM_LIMIT - 1024 - 512 - TBYTES - (long long)ks(H) * 16384;
    long long s = room / STAGE;
    return (int)(s > MAX_STAGES ? MAX_STAGES : s);
  }
  static size_t smem(int H) { return 1024 + (size_t)ks(H) * 16384 + TBYTES + (size_t)stages(H) * STAGE + 512; }
  static int ctas(int H, int B) { return (4 * H / NG) * ((B + ROWS - 1) / ROWS); }
  // TMEM staging of W reads the ring as up to stages*STAGE/16384 k-blocks per round
  static bool ok(int H, int B) {
    return H % (64 * KBOX) == 0 && (4 * H) % NG == 0 && stages(H) >= 2 && (stages(H) * STAGE) >= 16384 && B >= 1;
  }
};

CMT_D void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
CMT_D void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16
CMT_D void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
}  // namespace tm

template <int ROWS>
__global__ void __launch_bounds__(tm::THREADS, 1)
    lstm_fwd_tm(const __grid_constant__ CUtensorMap tmH0, const __grid_constant__ CUtensorMap tmW0,
                const __grid_constant__ CUtensorMap tmH1, const __grid_constant__ CUtensorMap tmW1,
                const LstmFwdMulti m) {
  using F = tm::Fwd<ROWS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int ch = (int)blockIdx.x >= m.split ? 1 : 0;
  const LstmFwdP p = ch ? m.c[1] : m.c[0];
  const int bid = ch ? (int)blockIdx.x - m.split : (int)blockIdx.x;
  const void* tmH = ch ? (const void*)&tmH1 : (const void*)&tmH0;
  const void* tmW = ch ? (const void*)&tmW1 : (const void*)&tmW0;

  const int KB = p.H / 64;
  const int KT = F::kt(p.H), KS = KB - KT;
  uint8_t* sW = smem;                                     // KS x 2 atoms [64 k][64 gc] (MN-major)
  float* sT = (float*)(smem + (size_t)KS * 16384);        // [ROWS][NG] transpose tile
  uint8_t* sB = (uint8_t*)sT + F::TBYTES;                 // stages x KBOX x [ROWS][64] (K-major)
  uint64_t* full = (uint64_t*)(sB + (size_t)p.stages * F::STAGE);
  uint64_t* empty = full + tm::MAX_STAGES;
  uint64_t* wfull = empty + tm::MAX_STAGES;
  uint64_t* sbar = wfull + 1;  // TMEM staging rounds
  uint64_t* tfull = sbar + 1;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nh = (p.B + ROWS - 1) / ROWS;
  const int half = bid % nh;
  const int n0 = (bid / nh) * tm::NG;
  const int u0 = n0 >> 2;
  const int r0 = half * ROWS;
  const int wrow0 = p.din;  // W_h rows start after the input rows of [W_x; W_h]
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(tmH);
    ptx::prefetch_tmap(tmW);
    for (int i = 0; i < p.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(wfull, 1);
    ptx::mbar_init(sbar, 1);
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty, tm::EPI);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, tm::TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tA = tmem + tm::D_COLS;  // W_h k-blocks [KS, KB) in TMEM

  // ---- load the W_h slice once: KS k-blocks to smem (async), KT k-blocks to
  // TMEM through the (still idle) stage ring ----
  if (threadIdx.x == 0 && KS > 0) {
    ptx::mbar_expect_tx(wfull, KS * 16384);
    for (int kb = 0; kb < KS; ++kb)
      for (int a = 0; a < 2; ++a)
        ptx::tma_load_2d(tmW, wfull, sW + kb * 16384 + a * 8192, n0 + a * 64, wrow0 + kb * 64);
  }
  {
    const int per = (p.stages * F::STAGE) / 16384;  // k-blocks per staging round
    int round = 0;
    for (int k0 = 0; k0 < KT; k0 += per, ++round) {
      const int nk = KT - k0 < per ? KT - k0 : per;
      if (threadIdx.x == 0) {
        ptx::mbar_expect_tx(sbar, nk * 16384);
        for (int i = 0; i < nk; ++i)
          for (int a = 0; a < 2; ++a)
            ptx::tma_load_2d(tmW, sbar, sB + i * 16384 + a * 8192, n0 + a * 64, wrow0 + (KS + k0 + i) * 64);
      }
      if (warp >= 4 && warp < 8) {
        ptx::mbar_wait(sbar, round & 1);
        const int mcol = (warp & 3) * 32 + lane;  // gate column = TMEM lane
        const uint8_t* atom = sB + (mcol >> 6) * 8192;
        const int mb = (mcol & 63) * 2;
        for (int i = 0; i < nk; ++i) {
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int k0r = 2 * c, k1r = 2 * c + 1;  // 128B swizzle: 16-byte chunk ^= (row & 7)
            const uint16_t lo = *(const uint16_t*)(atom + i * 16384 + k0r * 128 + ((((mb >> 4) ^ (k0r & 7)) << 4) | (mb & 15)));
            const uint16_t hi = *(const uint16_t*)(atom + i * 16384 + k1r * 128 + ((((mb >> 4) ^ (k1r & 7)) << 4) | (mb & 15)));
            r[c] = (uint32_t)lo | ((uint32_t)hi << 16);
          }
          tm::tmem_st32(tA + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((k0 + i) * 32), r);
        }
        tm::tmem_wait_st();
      }
      __syncthreads();  // the ring may be refilled
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();

  if (warp == 0) {
    // ===== producer: stream h_{t-1} k-blocks of this batch slice as their
    // two producer CTAs publish them (flag[kb * nh + half] reaches 2 s) =====
    int stage = 0;
    uint32_t phase = 0;
    const int nst = KB / F::KBOX;
    for (int s = 0; s < p.steps; ++s) {
      const int t = p.reverse ? p.steps - 1 - s : s;
      const int hrow = p.hrow0 + t * p.B + r0;
      const unsigned target = 2u * (unsigned)s;
      int issued = 0;
      SpinGuard guard;
      while (issued < nst) {
        unsigned ready = 0xffffffffu;
        if (s > 0) {
          const bool ok = lane >= KB || ptx::ld_acquire(p.flag + lane * nh + half) >= target;
          ready = __ballot_sync(0xffffffffu, ok);
          __syncwarp();
          if (ready != 0xffffffffu && __shfl_sync(0xffffffffu, lane == 0 ? (int)guard.expired(p.status) : 0, 0))
            ready = 0xffffffffu;  // wait budget exceeded: the step is reported failed
        }
        if (lane == 0) {
          if (s > 0) ptx::fence_proxy_async_global();
          while (issued < nst) {
            const unsigned need = ((1u << F::KBOX) - 1u) << (issued * F::KBOX);
            if ((ready & need) != need) break;
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            if (p.trace && bid == 0 && (issued == 0 || issued == nst - 1)) p.trace[s * 8 + (issued ? 4 : 0)] = gtimer();
            ptx::tma_load_3d(tmH, &full[stage], sB + stage * F::STAGE, 0, hrow, issued * F::KBOX);
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
      const uint32_t idesc_s = ptx::idesc_bf16(128, ROWS, 1, 0);  // A = W (smem, MN-major)
      const uint32_t idesc_t = ptx::idesc_bf16(128, ROWS, 0, 0);  // A = W (TMEM)
      if (KS > 0) ptx::mbar_wait(wfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t wbase = ptx::smem_u32(sW);
      for (int s = 0; s < p.steps; ++s) {
        ptx::mbar_wait(tempty, (s & 1) ^ 1);
        ptx::tc_fence_after();
        for (int kb0 = 0; kb0 < KB; kb0 += F::KBOX) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (p.trace && bid == 0 && (kb0 == 0 || kb0 + F::KBOX >= KB)) p.trace[s * 8 + (kb0 ? 6 : 5)] = gtimer();
          const uint32_t b0 = ptx::smem_u32(sB + stage * F::STAGE);
#pragma unroll
          for (int j = 0; j < F::KBOX; ++j) {
            const int kb = kb0 + j;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t bd = ptx::smem_desc_sw128(b0 + j * F::KBLK + kk * 32, 16, 1024);
              const uint32_t acc = (kb | kk) ? 1u : 0u;
              if (kb < KS) {
                const uint64_t ad = ptx::smem_desc_sw128(wbase + kb * 16384 + kk * 2048, 8192, 1024);
                ptx::umma_bf16(tmem, ad, bd, idesc_s, acc);
              } else {
                tm::umma_bf16_ts(tmem, tA + (uint32_t)((kb - KS) * 32 + kk * 8), bd, idesc_t, acc);
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
    // ===== epilogue: 8 warps.  Activation phase: warp e = warp - 4 reads TMEM
    // lane quadrant q = e & 3 (thread = gate column) for accumulator columns
    // (batch rows) [hc * ROWS/2, (hc + 1) * ROWS/2), hc = e >> 2.  Cell phase:
    // warp e / lane j = unit u0 + j for batch rows e + 8 i. =====
    constexpr int HB = ROWS / 2;  // batch rows per thread in the activation phase
    constexpr int NB = ROWS / 8;  // batch rows per thread in the cell phase
    const int e = warp - 4;
    const int q = e & 3, hc = e >> 2;
    const int mcol = q * 32 + lane;  // gate column n0 + mcol
    const int gate = mcol & 3;       // i, f, g, o (gate-interleaved columns)
    // act = a * tanh(sc * x) + o: sigmoid for i, f, o; tanh for g
    const float sc = gate == 2 ? 1.f : 0.5f, ao = gate == 2 ? 0.f : 0.5f, aa = gate == 2 ? 1.f : 0.5f;
    const long long H = p.H, H4 = 4LL * p.H;
    float c[NB], h[NB];
    {
      const int t0 = p.reverse ? p.steps - 1 : 0;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int b = r0 + e + 8 * i;
        const long long rr = ((long long)t0 * p.B + b) * H + u0 + lane;
        c[i] = b < p.B ? p.cprev[rr] : 0.f;
        h[i] = b < p.B ? __bfloat162float(p.hprev[rr]) : 0.f;
      }
    }
    float4* sT4 = (float4*)sT;
    for (int s = 0; s < p.steps; ++s) {
      const int t = p.reverse ? p.steps - 1 - s : s;
      const long long rbase = (long long)t * p.B + r0;  // token row of batch slot 0
      float x[HB];
#pragma unroll
      for (int k = 0; k < HB; ++k) {
        const int b = hc * HB + k;
        x[k] = (r0 + b < p.B) ? __ldg(p.ux + (rbase + b) * H4 + n0 + mcol) : 0.f;
      }
      float mk[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int b = e + 8 * i;
        mk[i] = (p.mask && r0 + b < p.B) ? __ldg(p.mask + rbase + b) : 1.f;
      }
      ptx::mbar_wait(tfull, s & 1);
      ptx::tc_fence_after();
      if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[s * 8 + 1] = gtimer();
      float v[HB];
#pragma unroll
      for (int c0 = 0; c0 < HB; c0 += 16) ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + hc * HB + c0, v + c0);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(tempty);
#pragma unroll
      for (int k = 0; k < HB; ++k) {
        const float a = fmaf(aa, ptx::tanh_fast(sc * (v[k] + x[k])), ao);
        v[k] = a;
        sT[(hc * HB + k) * tm::NG + mcol] = a;
      }
      ptx::named_bar_sync(1, 32 * tm::EPI);
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int b = e + 8 * i;
        const float4 g4 = sT4[b * tm::NU + lane];  // (i, f, g, o) of unit j at row b
        const float cn = fmaf(g4.y, c[i], g4.x * g4.z);
        const float tcn = ptx::tanh_fast(cn);
        const float hn = g4.w * tcn;
        if (p.mask) {
          h[i] = mk[i] * hn + (1.f - mk[i]) * h[i];
          c[i] = mk[i] * cn + (1.f - mk[i]) * c[i];
        } else {
          h[i] = hn;
          c[i] = cn;
        }
        mk[i] = tcn;  // reuse: tanh(c) cache
        if (r0 + b < p.B) p.y[(rbase + b) * H + u0 + lane] = __float2bfloat16_rn(h[i]);
      }
      if (p.trace && bid == 0 && threadIdx.x == 128) p.trace[s * 8 + 2] = gtimer();
      // publish h_t, then write the BPTT caches (the next step's sT writes are
      // ordered after this barrier, so the tile reads above are complete)
      ptx::named_bar_sync(1, 32 * tm::EPI);
      if (threadIdx.x == 128) {
        ptx::red_release_add(p.flag + (u0 >> 6) * nh + half, 1u);
        if (p.trace && bid == 0) p.trace[s * 8 + 3] = gtimer();
      }
#pragma unroll
      for (int k = 0; k < HB; ++k) {
        const int b = hc * HB + k;
        if (r0 + b < p.B) p.acts[(rbase + b) * H4 + n0 + mcol] = v[k];
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const int b = e + 8 * i;
        if (r0 + b < p.B) {
          p.tcache[(rbase + b) * H + u0 + lane] = mk[i];
          p.cst[(rbase + b) * H + u0 + lane] = c[i];
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, tm::TMEM_COLS);
  }
}

}  // namespace cmt
