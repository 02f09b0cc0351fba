// Batched beam search on the device.
//
// The reference translates one sentence at a time and runs decode_step once
// per live hypothesis (decoding.py:89-153, model.py:211-236).  Here every live
// hypothesis of every sentence of a batch is a row of one decoder step:
// rows = B sentences x K beam slots (row s*K + j = slot j of sentence s), so
// the step's products are GEMMs (the training path's tcgen05 kernels in bf16
// mode, the fp32 SIMT kernel in validation mode) and the whole hypothesis
// bookkeeping — top-K over live x V with the reference's tie order, EOS
// retirement into the finished pool, the exact stopping bound, the length cap —
// runs in beam_select_kernel, one warp per sentence.  The host reads one
// counter per step and, once every sentence is done, the back-pointers.
//
// Step t (kernels below in launch order; the GEMMs are issued by the engine):
//   beam_gather_kernel   parents' states -> layer inputs z_k[:, din:] and c_in
//   beam_embed_kernel    z_1[:, :E] = tgt_embed[token]
//   GEMM + beam_cell     U = z_k W_k + b;  (h, c) = cell(U, c_in) per layer
//   GEMM                 u = W_a^T h_top
//   beam_attention       alpha over the sentence's S source states, ctx
//   GEMMs                H_o = tanh(W_c^T [ctx; h_top]), Y = tanh(W_o^T H_o + b_o)
//   beam_topk_kernel     log_softmax row + its kk best (log-prob desc, token asc)
//   beam_select_kernel   the beam update of decoding.py:106-132
#pragma once
#include "common.cuh"

namespace cmt {
namespace bm {
constexpr int MAXK = 32;         // beam <= 32 (one warp lane per slot)
constexpr int TOPK_THREADS = 256;
constexpr int ATT_THREADS = 256;
}  // namespace bm

// per-sentence beam state (decoding.py:101-105)
struct BeamSent {
  int n_live;      // live hypotheses (slots 0..n_live-1)
  int done;        // search over for this sentence
  int t;           // decoder steps taken = tokens of every live hypothesis
  int nf;          // finished hypotheses so far (all of them, like the reference's list)
  int arrivals;    // arrival counter (ties of finished scores: earlier first)
  int max_len;     // cap_for(src_len) (>= 1)
  int trunc_slot;  // truncation fallback: the best live slot when nothing finished
  int pad;
  double best_fin; // max finished score
  double lp_cap;   // length_penalty(max_len)
};
// a finished hypothesis: EOS emitted at step t by live slot `parent` of step t-1
struct BeamFin {
  double score, logp;
  int arrival, t, parent, pad;
};

// z_k[r][din:din+H] = act(h of the parent row, layer k); cin[k][r] = its c.
// par[r] < 0: the encoder finals of the row's sentence (first step).
template <typename A>
__global__ void beam_gather_kernel(const float* __restrict__ h_src, const float* __restrict__ c_src,
                                   const float* __restrict__ fin_h, const float* __restrict__ fin_c,
                                   const int* __restrict__ par, int rows, int K, int B, int H, A* const* z,
                                   const int* zld, const int* zoff, float* __restrict__ cin) {
  const int r = blockIdx.x, k = blockIdx.y;
  const int p = par[r];
  const float* hs;
  const float* cs;
  if (p < 0) {
    const int s = r / K;
    hs = fin_h + ((long long)k * B + s) * H;
    cs = fin_c + ((long long)k * B + s) * H;
  } else {
    hs = h_src + ((long long)k * rows + p) * H;
    cs = c_src + ((long long)k * rows + p) * H;
  }
  A* zd = z[k] + (long long)r * zld[k] + zoff[k];
  float* cd = cin + ((long long)k * rows + r) * H;
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    zd[j] = from_f<A>(hs[j]);
    cd[j] = cs[j];
  }
}

// z[r][0:E] = table[ids[r]]
template <typename A>
__global__ void beam_embed_kernel(const A* __restrict__ table, const int* __restrict__ ids, int E, A* __restrict__ z,
                                  int ldz) {
  const int r = blockIdx.x;
  const A* src = table + (long long)ids[r] * E;
  A* d = z + (long long)r * ldz;
  for (int e = threadIdx.x; e < E; e += blockDim.x) d[e] = src[e];
}

// LSTM cell (layers.py:344-363) on gate-interleaved pre-activations U[r][4j+q]
// (bias folded by the GEMM): state (h, c) fp32, h also as the next product's input
template <typename A>
__global__ void beam_cell_kernel(const float* __restrict__ U, const float* __restrict__ cin, int H,
                                 float* __restrict__ h_out, float* __restrict__ c_out, A* __restrict__ xnext,
                                 int ldx) {
  const int r = blockIdx.x;
  for (int j = blockIdx.y * blockDim.x + threadIdx.x; j < H; j += gridDim.y * blockDim.x) {
    const float4 u = *(const float4*)(U + (long long)r * 4 * H + 4 * j);
    const float gi = sigmoidf_(u.x), gf = sigmoidf_(u.y), gg = tanhf(u.z), go = sigmoidf_(u.w);
    const float c = __fadd_rn(__fmul_rn(gf, cin[(long long)r * H + j]), __fmul_rn(gi, gg));
    const float h = __fmul_rn(go, tanhf(c));
    h_out[(long long)r * H + j] = h;
    c_out[(long long)r * H + j] = c;
    xnext[(long long)r * ldx + j] = from_f<A>(h);
  }
}

// Luong attention of row r over its sentence's source states (attend_values,
// attention.py:235-250): scores_s = Hs_s . u_r, masked softmax over s (masked
// positions exactly 0 by predicate, the reference's additive -1e9 makes them
// exp(-1e9)=0 as well), ctx_r = sum_s alpha_s Hs_s -> zc[r][0:H].
// Hs rows are the encoder top output, row s*B + b (b = the row's sentence).
template <typename A>
__global__ void __launch_bounds__(bm::ATT_THREADS) beam_attention_kernel(const A* __restrict__ hs, int S, int B, int H,
                                                                         const float* __restrict__ smask,
                                                                         const float* __restrict__ u, int K,
                                                                         A* __restrict__ zc, int ldzc) {
  extern __shared__ float sc[];  // [S]
  __shared__ float red[32];
  const int r = blockIdx.x, b = r / K;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const float* ur = u + (long long)r * H;
  for (int s = warp; s < S; s += nw) {
    const A* hr = hs + ((long long)s * B + b) * H;
    float a = 0.f;
    for (int h = lane; h < H; h += 32) a = fmaf(to_f<A>(hr[h]), ur[h], a);
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) sc[s] = a;
  }
  __syncthreads();
  if (warp == 0) {
    float m = -INFINITY;
    for (int s = lane; s < S; s += 32)
      if (smask[(long long)s * B + b] != 0.f) m = fmaxf(m, sc[s]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float z = 0.f;
    for (int s = lane; s < S; s += 32) {
      const float e = smask[(long long)s * B + b] != 0.f ? expf(sc[s] - m) : 0.f;
      sc[s] = e;
      z += e;
    }
    for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (lane == 0) red[0] = z;
  }
  __syncthreads();
  const float z = red[0];
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    float c = 0.f;
    for (int s = 0; s < S; ++s) {
      const float a = sc[s] / z;
      c = fmaf(a, to_f<A>(hs[((long long)s * B + b) * H + h]), c);
    }
    zc[(long long)r * ldzc + h] = from_f<A>(c);
  }
}

// (lp, tok) order of the candidates: log-prob descending, token ascending
CMT_D bool beam_better(float a, int ta, float b, int tb) { return a > b || (a == b && ta < tb); }

// Insert (v, t) into the warp's sorted list (lane i holds entry i, kk entries).
CMT_D void warp_list_insert(float& lv, int& lt, int kk, float v, int t) {
  const int lane = threadIdx.x & 31;
  const unsigned ahead = __ballot_sync(0xffffffffu, lane < kk && beam_better(lv, lt, v, t));
  const int pos = __popc(ahead);
  const float uv = __shfl_up_sync(0xffffffffu, lv, 1);
  const int ut = __shfl_up_sync(0xffffffffu, lt, 1);
  if (pos < kk) {
    if (lane == pos) { lv = v; lt = t; }
    else if (lane > pos && lane < kk) { lv = uv; lt = ut; }
  }
}

// log_softmax_columns (tensor.py:146-151) of row r and its kk best entries in
// the order (log-prob desc, token asc).  Rows of finished sentences and
// slots beyond the live count are skipped.
__global__ void __launch_bounds__(bm::TOPK_THREADS) beam_topk_kernel(const float* __restrict__ Y, int V, int kk, int K,
                                                                     const BeamSent* __restrict__ sent,
                                                                     float* __restrict__ top_val,
                                                                     int* __restrict__ top_tok,
                                                                     int* __restrict__ status) {
  __shared__ float rm[32], rz[32];
  __shared__ float wl[32 * bm::MAXK];
  __shared__ int wt[32 * bm::MAXK];
  const int r = blockIdx.x;
  const BeamSent st = sent[r / K];
  if (st.done || (r % K) >= st.n_live) return;
  const float* y = Y + (long long)r * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // pass 1: max and sum of exponentials (running rescale)
  float m = -INFINITY, z = 0.f;
  bool bad = false;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float x = y[v];
    bad |= !isfinite(x);
    if (x > m) { z = z * expf(m - x) + 1.f; m = x; }
    else z += expf(x - m);
  }
  for (int o = 16; o; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o), oz = __shfl_xor_sync(0xffffffffu, z, o);
    const float nm = fmaxf(m, om);
    z = (m == -INFINITY ? 0.f : z * expf(m - nm)) + (om == -INFINITY ? 0.f : oz * expf(om - nm));
    m = nm;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_LOGITS);
  if (lane == 0) { rm[warp] = m; rz[warp] = z; }
  __syncthreads();
  float mx = -INFINITY;
  for (int w = 0; w < nw; ++w) mx = fmaxf(mx, rm[w]);
  float zs = 0.f;
  for (int w = 0; w < nw; ++w) zs += rm[w] == -INFINITY ? 0.f : rz[w] * expf(rm[w] - mx);
  const float lse = logf(zs);
  // pass 2: per-warp sorted top-kk lists, then warp 0 merges them
  float lv = -INFINITY;
  int lt = 0x7fffffff;
  const int per = (V + nw - 1) / nw;
  const int v0 = warp * per, v1 = min(V, v0 + per);
  for (int base = v0; base < v1; base += 32) {
    const int v = base + lane;
    const float x = v < v1 ? (y[v] - mx) - lse : -INFINITY;
    const float kv = __shfl_sync(0xffffffffu, lv, kk - 1);
    const int kt = __shfl_sync(0xffffffffu, lt, kk - 1);
    unsigned cand = __ballot_sync(0xffffffffu, v < v1 && beam_better(x, v, kv, kt));
    while (cand) {
      const int src = __ffs(cand) - 1;
      cand &= cand - 1;
      const float cv = __shfl_sync(0xffffffffu, x, src);
      warp_list_insert(lv, lt, kk, cv, base + src);
    }
  }
  if (lane < kk) { wl[warp * bm::MAXK + lane] = lv; wt[warp * bm::MAXK + lane] = lt; }
  __syncthreads();
  if (warp != 0) return;
  for (int w = 1; w < nw; ++w)
    for (int i = 0; i < kk; ++i) {
      const float cv = wl[w * bm::MAXK + i];
      const int ct = wt[w * bm::MAXK + i];
      const float kv = __shfl_sync(0xffffffffu, lv, kk - 1);
      const int kt = __shfl_sync(0xffffffffu, lt, kk - 1);
      if (!beam_better(cv, ct, kv, kt)) break;  // the warp's list is sorted: the rest is worse
      warp_list_insert(lv, lt, kk, cv, ct);
    }
  if (lane < kk) {
    top_val[(long long)r * kk + lane] = lv;
    top_tok[(long long)r * kk + lane] = lt;
  }
}

// The beam update of one sentence (decoding.py:106-132), one warp:
//   candidates: live slot j's log-prob (double) + its row's kk best log-probs;
//   the beam best in the order (score desc, slot asc, token asc) by a K-way
//   merge of the per-slot lists (lane j = slot j);
//   EOS children retire into the finished pool (score = log_prob / lp(t+1),
//   kept sorted by (score desc, arrival asc), the best nb of them), the others
//   become the new live slots in order;
//   stop when no live slot remains, when at least `beam` have finished and the
//   best live bound max(log_prob) / lp(max_len) cannot beat the best finished
//   score, or at the length cap.  lptab[n] = length_penalty(n) from the host
//   (bit-identical to the reference's ((5 + n) / 6) ** alpha).
__global__ void beam_select_kernel(BeamSent* __restrict__ sent, double* __restrict__ live_lp,
                                   const float* __restrict__ top_val, const int* __restrict__ top_tok, int K, int kk,
                                   int beam, int2* __restrict__ bp, int Tmax, BeamFin* __restrict__ fin, int nb,
                                   const double* __restrict__ lptab, int* __restrict__ ids, int* __restrict__ par,
                                   int* __restrict__ nactive, int eos) {
  const int s = blockIdx.x, lane = threadIdx.x;
  BeamSent st = sent[s];
  if (st.done) return;
  const int n = st.n_live, t = st.t;
  const long long row = (long long)s * K + lane;
  const double base = lane < n ? live_lp[row] : 0.0;
  int p = 0;
  // chosen children, in order (held by lane i = i-th choice)
  double cs = 0.0;
  int cj = -1, ctok = -1;
  int nchosen = 0;
  for (int i = 0; i < beam; ++i) {
    const bool has = lane < n && p < kk;
    const double sc = has ? base + (double)top_val[row * kk + p] : -INFINITY;
    // warp argmax: score desc, then lane (slot) asc
    double bs = sc;
    int bl = has ? lane : 64;
    for (int o = 16; o; o >>= 1) {
      const double os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (ol < 64 && (bl == 64 || os > bs || (os == bs && ol < bl))) { bs = os; bl = ol; }
    }
    if (bl == 64) break;  // fewer than beam candidates (live x V < beam)
    const int tok = __shfl_sync(0xffffffffu, lane == bl ? top_tok[row * kk + p] : 0, bl);
    if (lane == i) { cs = bs; cj = bl; ctok = tok; }
    if (lane == bl) ++p;
    ++nchosen;
  }
  // lane 0 walks the choices in order (values gathered through shared memory)
  __shared__ double s_sc[bm::MAXK];
  __shared__ int s_j[bm::MAXK], s_tok[bm::MAXK];
  if (lane < nchosen) { s_sc[lane] = cs; s_j[lane] = cj; s_tok[lane] = ctok; }
  __syncwarp();
  if (lane != 0) return;
  int n_new = 0;
  double best_live = -INFINITY;
  BeamFin* pool = fin + (long long)s * nb;
  for (int i = 0; i < nchosen; ++i) {
    const double sc = s_sc[i];
    const int j = s_j[i], tok = s_tok[i];
    if (tok == eos) {
      BeamFin f;
      f.score = sc / lptab[t + 1];
      f.logp = sc;
      f.arrival = st.arrivals++;
      f.t = t;
      f.parent = j;
      f.pad = 0;
      const int have = min(st.nf, nb);
      // insertion position in (score desc, arrival asc): after every entry with score >= f.score
      int pos = have;
      while (pos > 0 && pool[pos - 1].score < f.score) --pos;
      if (pos < nb) {
        for (int q = min(have, nb - 1); q > pos; --q) pool[q] = pool[q - 1];
        pool[pos] = f;
      }
      st.nf++;
      st.best_fin = fmax(st.best_fin, f.score);
    } else {
      const int m = n_new++;
      live_lp[(long long)s * K + m] = sc;
      bp[((long long)s * Tmax + t) * K + m] = make_int2(j, tok);
      ids[(long long)s * K + m] = tok;
      par[(long long)s * K + m] = s * K + j;
      best_live = fmax(best_live, sc);
    }
  }
  st.t = t + 1;
  st.n_live = n_new;
  if (n_new == 0) st.done = 1;
  else if (st.nf >= beam && best_live / st.lp_cap <= st.best_fin) st.done = 1;
  else if (st.t >= st.max_len) st.done = 1;
  if (st.done && st.nf == 0) {  // truncation: the first live slot of maximal log-prob
    int b = 0;
    for (int m = 1; m < n_new; ++m)
      if (live_lp[(long long)s * K + m] > live_lp[(long long)s * K + b]) b = m;
    st.trunc_slot = b;
  }
  if (!st.done) atomicAdd(nactive, 1);
  sent[s] = st;
}

}  // namespace cmt
