// Parameters shared by the persistent recurrent kernels (lstm_multi.cuh,
// lstm_tm.cuh) and the bounded wait on the cross-CTA readiness flags.
// Reference semantics: layers.py:344-395 (cell forward/backward),
// layers.py:440-493 (masked scan / BPTT).
#pragma once
#include "ptx.cuh"

namespace cmt {

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
  int* status;          // step status word (ST_HANG on a wait timeout)
  int steps, B, H, din, reverse;
  int hrow0;            // row of h_{-1}(t=0) in the Yext tensor map
  int stages;
  unsigned long long* trace;  // debug: per-step phase timestamps of CTA 0 (or null)
};

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
  int* status;           // step status word (ST_HANG on a wait timeout)
  int steps, B, H, din, reverse;
  int stages;
  unsigned long long* trace;
};

CMT_D unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Hang guard of the flag polls.  A scan step waits for k-blocks that other
// CTAs publish; that needs every CTA of the launch resident, which the
// cooperative launch guarantees in normal runs.  If a wait ever exceeds the
// budget (~0.5 s, 5e4x a step; e.g. CTAs serialised by a profiler's replay) the
// waiter raises ST_HANG in the step status, and every later wait of the step
// sees it and falls through: the launch ends with wrong numbers and the step
// reports an internal error instead of hanging the device.
struct SpinGuard {
  long long t0 = 0;
  unsigned it = 0;
  // call while still waiting; true = give up
  CMT_D bool expired(int* status) {
    if ((++it & 63u) != 0) return false;
    const long long now = clock64();
    if (t0 == 0) { t0 = now; return false; }
    if (*(volatile int*)status & ST_HANG) return true;
    if (now - t0 > (1LL << 30)) {
      atomicOr(status, ST_HANG);
      return true;
    }
    return false;
  }
};

}  // namespace cmt
