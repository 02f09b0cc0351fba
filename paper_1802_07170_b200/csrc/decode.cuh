// GPU translation step: the reference's INFER-mode
// decode_step (model.py:211-236) for the n live hypotheses of one sentence as
// the rows of small batched products.  At n <= 16 every product is a
// weight-streaming GEMV (each weight byte is read once per step), so these are
// bandwidth kernels over the bf16 shadow (or fp32 masters in validation mode),
// fp32 arithmetic throughout.  The encoder side reuses the training forward.
#pragma once
#include "common.cuh"

namespace cmt {
namespace dec {
constexpr int ROWS = 16;       // hypotheses per GEMV pass (grid.z covers more)
constexpr int GV_THREADS = 128;
constexpr int GV_COLS = 2 * GV_THREADS;  // output columns per CTA (2 per thread)
constexpr int KCH = 128;       // K chunk per CTA (split-K partials)
constexpr int TOPK_THREADS = 1024;
constexpr int MAXK = 32;
}  // namespace dec

template <typename T>
CMT_D float2 ld2f(const T* p);
template <>
CMT_D float2 ld2f<float>(const float* p) { return *(const float2*)p; }
template <>
CMT_D float2 ld2f<bf16>(const bf16* p) { return __bfloat1622float2(*(const __nv_bfloat162*)p); }

// part[ks][i][j] = sum_{k in chunk ks} Z[i][k] W[k][j]   (rows i of this z-slice)
template <typename T>
__global__ void __launch_bounds__(dec::GV_THREADS) dec_gemv_partial(const float* __restrict__ Z, int ldz, int n, int K,
                                                                   const T* __restrict__ W, long long ldw, int N,
                                                                   float* __restrict__ part) {
  __shared__ float zs[dec::ROWS][dec::KCH];
  const int i0 = blockIdx.z * dec::ROWS, nr = min(dec::ROWS, n - i0);
  const int k0 = blockIdx.y * dec::KCH, nk = min(dec::KCH, K - k0);
  for (int x = threadIdx.x; x < dec::ROWS * dec::KCH; x += blockDim.x) {
    const int i = x / dec::KCH, k = x % dec::KCH;
    zs[i][k] = (i < nr && k < nk) ? Z[(long long)(i0 + i) * ldz + k0 + k] : 0.f;
  }
  __syncthreads();
  const int j = blockIdx.x * dec::GV_COLS + 2 * threadIdx.x;
  if (j >= N) return;
  const bool two = j + 1 < N;
  float a0[dec::ROWS], a1[dec::ROWS];
#pragma unroll
  for (int i = 0; i < dec::ROWS; ++i) a0[i] = a1[i] = 0.f;
  const T* wp = W + (long long)k0 * ldw + j;
  const bool vec = two && ((ldw & 1) == 0) && ((j & 1) == 0);
#pragma unroll 4
  for (int k = 0; k < nk; ++k) {
    float2 w;
    if (vec) w = ld2f<T>(wp + (long long)k * ldw);
    else w = make_float2(to_f<T>(wp[(long long)k * ldw]), two ? to_f<T>(wp[(long long)k * ldw + 1]) : 0.f);
#pragma unroll
    for (int i = 0; i < dec::ROWS; ++i) {
      a0[i] = fmaf(zs[i][k], w.x, a0[i]);
      a1[i] = fmaf(zs[i][k], w.y, a1[i]);
    }
  }
  float* pp = part + ((long long)blockIdx.y * n + i0) * N + j;
  for (int i = 0; i < nr; ++i) {
    pp[(long long)i * N] = a0[i];
    if (two) pp[(long long)i * N + 1] = a1[i];
  }
}

// Bandwidth-shaped variant: CTA = 128 output columns x one K chunk; its 8
// warps split the chunk, lane = 4 adjacent columns (8-byte bf16 / 16-byte fp32
// weight loads, a warp reads 256 / 512 contiguous bytes per weight row), all
// n <= 16 rows accumulate in registers; the 8 warp partials are added in smem
// in warp order, so part[ks][i][j] is deterministic.
constexpr int GV2_THREADS = 256, GV2_COLS = 128, GV2_KCH = 256;
constexpr size_t GV2_SMEM = sizeof(float) * (dec::ROWS * GV2_KCH + (GV2_THREADS / 32) * dec::ROWS * (GV2_COLS + 4));
// Inputs come as two column segments (Z1: K1 columns, Z2: K2 columns; K =
// K1 + K2), so [x; h] and [ctx; h] need no concatenation copies.  The last CTA
// of a column block (atomic ticket, reset by it) adds the K-chunk partials in
// chunk order, applies bias and activation and writes Y: one launch per product.
template <typename T>
__global__ void __launch_bounds__(GV2_THREADS) dec_gemv2(const float* __restrict__ Z1, int ld1, int K1,
                                                         const float* __restrict__ Z2, int ld2, int K2, int n,
                                                         const T* __restrict__ W, long long ldw, int N,
                                                         float* __restrict__ part, unsigned* __restrict__ ticket,
                                                         const float* __restrict__ bias, int act, float* __restrict__ Y,
                                                         int ldy) {
  const int K = K1 + K2;
  extern __shared__ float gv2_smem[];  // zs [ROWS][KCH], then red [warps][ROWS][COLS + 4]
  float(*zs)[GV2_KCH] = (float(*)[GV2_KCH])gv2_smem;
  float(*red)[dec::ROWS][GV2_COLS + 4] = (float(*)[dec::ROWS][GV2_COLS + 4])(gv2_smem + dec::ROWS * GV2_KCH);
  const int k0 = blockIdx.y * GV2_KCH, nk = min(GV2_KCH, K - k0);
  for (int x = threadIdx.x; x < dec::ROWS * GV2_KCH; x += blockDim.x) {
    const int i = x / GV2_KCH, k = x % GV2_KCH, kg = k0 + k;
    zs[i][k] = (i < n && k < nk) ? (kg < K1 ? Z1[(long long)i * ld1 + kg] : Z2[(long long)i * ld2 + kg - K1]) : 0.f;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * GV2_COLS + lane * 4;
  constexpr int KW = GV2_KCH / (GV2_THREADS / 32);  // k rows per warp
  float acc[dec::ROWS][4];
#pragma unroll
  for (int i = 0; i < dec::ROWS; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  if (c < N) {
    const bool full4 = c + 3 < N && (ldw & 3) == 0;
    const int kb = warp * KW, ke = min(nk, kb + KW);
#pragma unroll 4
    for (int k = kb; k < ke; ++k) {
      const T* wp = W + (long long)(k0 + k) * ldw + c;
      float w[4];
      if (full4) {
        if constexpr (sizeof(T) == 2) {
          const uint2 q = __ldg((const uint2*)wp);
          const float2 a = __bfloat1622float2(*(const __nv_bfloat162*)&q.x);
          const float2 b = __bfloat1622float2(*(const __nv_bfloat162*)&q.y);
          w[0] = a.x; w[1] = a.y; w[2] = b.x; w[3] = b.y;
        } else {
          const float4 q = __ldg((const float4*)wp);
          w[0] = q.x; w[1] = q.y; w[2] = q.z; w[3] = q.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = c + j < N ? to_f<T>(wp[j]) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < dec::ROWS; ++i) {
        const float z = zs[i][k];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(z, w[j], acc[i][j]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < dec::ROWS; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) red[warp][i][lane * 4 + j] = acc[i][j];
  __syncthreads();
  for (int x = threadIdx.x; x < n * GV2_COLS; x += blockDim.x) {
    const int i = x / GV2_COLS, cc = x % GV2_COLS;
    const int col = blockIdx.x * GV2_COLS + cc;
    if (col >= N) continue;
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < GV2_THREADS / 32; ++w) t += red[w][i][cc];
    part[((long long)blockIdx.y * n + i) * N + col] = t;
  }
  __threadfence();
  __shared__ unsigned last;
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket + blockIdx.x, 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int x = threadIdx.x; x < n * GV2_COLS; x += blockDim.x) {
    const int i = x / GV2_COLS, col = blockIdx.x * GV2_COLS + x % GV2_COLS;
    if (col >= N) continue;
    float t = 0.f;
    for (int q = 0; q < (int)gridDim.y; ++q) t += __ldcg(part + ((long long)q * n + i) * N + col);
    if (bias) t += bias[col];
    if (act == 1) t = tanhf(t);
    Y[(long long)i * ldy + col] = t;
  }
  if (threadIdx.x == 0) ticket[blockIdx.x] = 0u;
}

// Y[i][j] = act(sum_ks part[ks][i][j] + bias[j]); act 1 = tanh
__global__ void dec_gemv_final(const float* __restrict__ part, int ks, int n, int N, const float* __restrict__ bias,
                               int act, float* __restrict__ Y, int ldy) {
  const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= (long long)n * N) return;
  const int i = (int)(x / N), j = (int)(x % N);
  float s = 0.f;
  for (int c = 0; c < ks; ++c) s += part[((long long)c * n + i) * N + j];
  if (bias) s += bias[j];
  if (act == 1) s = tanhf(s);
  Y[(long long)i * ldy + j] = s;
}

// z[i][0:E] = table[ids[i]]
template <typename T>
__global__ void dec_embed(const T* __restrict__ table, const int* __restrict__ ids, int E, float* __restrict__ z,
                          int ldz) {
  const int i = blockIdx.x;
  const T* r = table + (long long)ids[i] * E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) z[(long long)i * ldz + e] = to_f<T>(r[e]);
}

// dst[l][i][:] = parent ? src[l][parent[i]][:] : fin[l][:]   (h and c of every decoder layer)
__global__ void dec_gather_states(const float* __restrict__ src_h, const float* __restrict__ src_c,
                                  const float* __restrict__ fin_h, const float* __restrict__ fin_c,
                                  const int* __restrict__ parent, int n, int H, long long lstride,
                                  float* __restrict__ dst_h, float* __restrict__ dst_c) {
  const int i = blockIdx.x, l = blockIdx.y;
  const float* sh = parent ? src_h + l * lstride + (long long)parent[i] * H : fin_h + (long long)l * H;
  const float* sc = parent ? src_c + l * lstride + (long long)parent[i] * H : fin_c + (long long)l * H;
  float* dh = dst_h + l * lstride + (long long)i * H;
  float* dc = dst_c + l * lstride + (long long)i * H;
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    dh[j] = sh[j];
    dc[j] = sc[j];
  }
}

__global__ void dec_copy_rows(const float* __restrict__ s, int lds, float* __restrict__ d, int ldd, int cols) {
  const int i = blockIdx.x;
  for (int j = threadIdx.x; j < cols; j += blockDim.x) d[(long long)i * ldd + j] = s[(long long)i * lds + j];
}

CMT_D float dec_sigmoid(float x) {  // stable split form (tensor.py:165-172)
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}
// LSTM cell (layers.py:344-363) on gate-interleaved pre-activations U[i][4j+q]
__global__ void dec_lstm_cell(const float* __restrict__ U, const float* __restrict__ c_in, int H,
                              float* __restrict__ h_out, float* __restrict__ c_out, float* __restrict__ z_next,
                              int ldz) {
  const int i = blockIdx.x;
  for (int j = blockIdx.y * blockDim.x + threadIdx.x; j < H; j += gridDim.y * blockDim.x) {
    const float4 u = *(const float4*)(U + ((long long)i * H + j) * 4);
    const float ig = dec_sigmoid(u.x), fg = dec_sigmoid(u.y), gg = tanhf(u.z), og = dec_sigmoid(u.w);
    const float c = fg * c_in[(long long)i * H + j] + ig * gg;
    const float h = og * tanhf(c);
    c_out[(long long)i * H + j] = c;
    h_out[(long long)i * H + j] = h;
    if (z_next) z_next[(long long)i * ldz + j] = h;
  }
}

// Luong attention of query row i over the S encoder states (attend_values,
// attention.py:235-250; one sentence, no padding): ctx[i] -> z2[i][0:H]
__global__ void dec_attention(const float* __restrict__ hs, int S, int H, const float* __restrict__ u,
                              float* __restrict__ z2, int ldz) {
  extern __shared__ float sc[];  // [S]
  __shared__ float red[32];
  const int i = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int s = warp; s < S; s += nw) {  // score_product: a warp per source position
    float a = 0.f;
    for (int h = lane; h < H; h += 32) a = fmaf(hs[(long long)s * H + h], u[(long long)i * H + h], a);
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) sc[s] = a;
  }
  __syncthreads();
  if (warp == 0) {  // softmax_columns (tensor.py:137-143)
    float m = -INFINITY;
    for (int s = lane; s < S; s += 32) m = fmaxf(m, sc[s]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float t = 0.f;
    for (int s = lane; s < S; s += 32) {
      const float e = expf(sc[s] - m);
      sc[s] = e;
      t += e;
    }
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.f / red[0];
  for (int h = threadIdx.x; h < H; h += blockDim.x) {  // weighted_sum
    float a = 0.f;
    for (int s = 0; s < S; ++s) a = fmaf(hs[(long long)s * H + h], sc[s] * inv, a);
    z2[(long long)i * ldz + h] = a;
  }
}

// log_softmax_columns (tensor.py:146-151) of row i and its k best entries in
// the order (log-prob descending, token ascending): round r takes the best
// entry strictly after round r-1's winner in that total order.
__global__ void __launch_bounds__(dec::TOPK_THREADS) dec_logsoftmax_topk(const float* __restrict__ Y, int V, int k,
                                                                       float* __restrict__ top_val,
                                                                       int* __restrict__ top_tok,
                                                                       int* __restrict__ status) {
  __shared__ float rv[32];
  __shared__ int ri[32];
  __shared__ float bc[2];
  const int i = blockIdx.x;
  const float* y = Y + (long long)i * V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float m = -INFINITY;
  bool bad = false;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    bad |= !isfinite(y[v]);
    m = fmaxf(m, y[v]);
  }
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, ST_LOGITS);
  if (lane == 0) rv[warp] = m;
  __syncthreads();
  if (warp == 0) {
    float x = lane < (int)(blockDim.x >> 5) ? rv[lane] : -INFINITY;
    for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) bc[0] = x;
  }
  __syncthreads();
  const float mx = bc[0];
  float t = 0.f;
  for (int v = threadIdx.x; v < V; v += blockDim.x) t += expf(y[v] - mx);
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  if (lane == 0) rv[warp] = t;
  __syncthreads();
  if (warp == 0) {
    float x = lane < (int)(blockDim.x >> 5) ? rv[lane] : 0.f;
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) bc[1] = logf(x);
  }
  __syncthreads();
  const float lse = bc[1];
  // top-k on the raw values (log-prob = y - max - lse is monotone in y)
  float pv = INFINITY;
  int pi = -1;
  for (int r = 0; r < k; ++r) {
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
      const float x = y[v];
      const bool after = (x < pv) || (x == pv && v > pi);  // strictly after the previous winner
      const bool better = (x > bv) || (x == bv && v < bi);
      if (after && better) { bv = x; bi = v; }
    }
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    __syncthreads();
    if (lane == 0) { rv[warp] = bv; ri[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      bv = lane < (int)(blockDim.x >> 5) ? rv[lane] : -INFINITY;
      bi = lane < (int)(blockDim.x >> 5) ? ri[lane] : 0x7fffffff;
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) {
        rv[0] = bv;
        ri[0] = bi;
        top_val[(long long)i * k + r] = (bv - mx) - lse;
        top_tok[(long long)i * k + r] = bi;
      }
    }
    __syncthreads();
    pv = rv[0];
    pi = ri[0];
  }
}

}  // namespace cmt
