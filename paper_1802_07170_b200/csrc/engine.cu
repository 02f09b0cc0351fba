// CytonMT B200 train-step engine: device memory layout, step orchestration
// and the C ABI declared in include/cytonmt_b200.h.
//
// The step implemented is reference training.py:145-159 (see SURVEY §8(a)
// "Exact step semantics").  Layout in HBM:
//   activations token-major [n][dim], n = t*B + b (the reference's (dim, N)
//   C-order arrays read column-wise);  LSTM weights of a layer merged into
//   one [Din+H][4H] matrix with gate-interleaved columns (4j+q = gate q of
//   unit j) so any 32-column GEMM chunk holds whole units for the fused cell
//   epilogues; every other weight keeps the reference's (dim_in, dim_out)
//   layout.  Dense params / grads / bf16 shadows live in three parallel
//   arenas (identical offsets) so clip-norm + SGD + shadow refresh are single
//   passes; embedding grads are row-compact (only touched rows exist).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_profiler_api.h>
#include <dlfcn.h>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "../../include/cytonmt_b200.h"
#include "gemm.cuh"
#include "kernels.cuh"
#include "lstm_multi.cuh"
#include "lstm_tm.cuh"
#include "attention.cuh"
#include "attention_tc.cuh"
#include "decode.cuh"

namespace cmt {
unsigned long long g_launches = 0;

// ---------------------------------------------------------------------------
// TMA descriptor creation (driver entry point fetched through the runtime)
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CMT_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Error(CMT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// bf16 2-D map: dim0 contiguous (extent d0), dim1 (extent d1, stride ld elems)
static void make_map(CUtensorMap* m, const void* ptr, long long d0, long long d1, long long ld, int box0, int box1) {
  if (((uintptr_t)ptr & 15) || ((ld * 2) & 15))
    throw Error(CMT_ERR_SHAPE, "bf16 GEMM operand not 16-byte aligned (dims must be multiples of 8 in bf16 mode)");
  cuuint64_t gdim[2] = {(cuuint64_t)d0, (cuuint64_t)d1};
  cuuint64_t gstr[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), gdim, gstr, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(CMT_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

// Epilogue output map for the TMA-store GEMM epilogue: C [rows][cols] (row
// stride ld elements), box 32 x 32, fp32 rows 128 B (SWIZZLE_128B) or bf16
// rows 64 B (SWIZZLE_64B), matching the smem staging layout in gemm.cuh.
static bool c_map_ok(const void* ptr, long long ld, bool bf16) {
  return !(((uintptr_t)ptr & 15) || ((ld * (bf16 ? 2 : 4)) & 15));
}
static void make_map_c(CUtensorMap* m, const void* ptr, long long cols, long long rows, long long ld, bool bf16) {
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstr[1] = {(cuuint64_t)(ld * (bf16 ? 2 : 4))};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                            const_cast<void*>(ptr), gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(CMT_ERR_CUDA, "cuTensorMapEncodeTiled (C) failed: " + std::to_string((int)r));
}

// bf16 3-D map over a row-major [rows][cols] matrix viewed as {64, rows, cols/64}
// (strides {ld*2, 128 B}): one TMA fetches `box2` consecutive 64-column blocks
// of `box1` rows into smem as box2 stacked [box1][64] 128B-swizzled tiles.
static void make_map_kblocks(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int box1,
                             int box2) {
  if (((uintptr_t)ptr & 15) || ((ld * 2) & 15) || (cols % 64))
    throw Error(CMT_ERR_SHAPE, "k-block TMA map needs 16-byte aligned rows and cols % 64 == 0");
  cuuint64_t gdim[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
  cuuint64_t gstr[2] = {(cuuint64_t)(ld * 2), 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box1, (cuuint32_t)box2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), gdim, gstr, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(CMT_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed: " + std::to_string((int)r));
}

// ---------------------------------------------------------------------------
// NCCL, loaded at runtime (the process may already hold torch's libnccl.so.2)
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  int (*get_unique_id)(void*) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  const char* (*get_error)(int) = nullptr;
  void load() {
    if (h) return;
    // the NCCL already in the process (torch's) if any; otherwise a private
    // copy: RTLD_LOCAL keeps its symbols from binding a later torch import
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) throw Error(CMT_ERR_CUDA, std::string("cannot load libnccl.so.2: ") + dlerror());
    get_unique_id = (int (*)(void*))dlsym(h, "ncclGetUniqueId");
    all_reduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclAllReduce");
    comm_destroy = (int (*)(void*))dlsym(h, "ncclCommDestroy");
    get_error = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    if (!get_unique_id || !all_reduce || !comm_destroy) throw Error(CMT_ERR_CUDA, "libnccl.so.2 lacks symbols");
  }
};
static NcclApi g_nccl;
struct NcclUid { char internal[128]; };
enum { NCCL_INT32 = 2, NCCL_FLOAT32 = 7, NCCL_FLOAT64 = 8, NCCL_SUM = 0, NCCL_MAX = 2 };

struct Mat {
  const void* p;
  long long ld;
  int mn;  // 1: MN-major (m/n contiguous), 0: K-major
};

static int g_num_sms = 148;
// Recurrent scans are cooperative launches (every CTA co-resident: the steps
// wait on each other's readiness flags).  Under a profiler's kernel replay
// (an injection library is attached: ncu sets NV_NSIGHT_INJECTION_*) the cluster
// kernels fail as cooperative launches (LaunchFailed), and each launch runs
// alone on an idle device anyway, so the attribute is dropped there
// (CMT_COOP=0/1 overrides).  A launch that is ever not co-resident cannot hang:
// the flag waits are bounded (lstm_common.cuh SpinGuard) and fail the step.
static int coop_default() {
  if (const char* v = getenv("CMT_COOP")) return atoi(v) != 0;
  const bool profiler = getenv("CUDA_INJECTION64_PATH") || getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") ||
                        getenv("NV_TPS_LAUNCH_TOKEN");
  return profiler ? 0 : 1;
}
static int g_coop = coop_default();
static int g_grid_cap = 0;  // > 0: persistent GEMMs use at most this many CTAs (work beside a running scan)
constexpr int FLAG_STRIDE = 128;  // step counters per scan (per-k-block readiness flags)

// ---- kernel timeline (debug option "timeline"): an event after every launch
// on the engine stream; consecutive event deltas are the per-launch device
// times measured in the real step, not under a profiler ----
struct Timeline {
  bool on = false;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  cudaEvent_t start = nullptr;
};
static Timeline g_tl;
static void tl_mark(cudaStream_t st, const std::string& label) {
  if (!g_tl.on) return;
  cudaEvent_t ev;
  CMT_CUDA(cudaEventCreate(&ev));
  CMT_CUDA(cudaEventRecord(ev, st));
  g_tl.marks.push_back({label, ev});
}
static std::string gemm_label(int M, int N, int K, int BN, int CG) {
  return "gemm " + std::to_string(M) + "x" + std::to_string(N) + "x" + std::to_string(K) + " t" + std::to_string(BN) +
         (CG == 2 ? "x2" : "");
}

static int g_gemm_opt = 0;  // option: bit 0 natural K order, bit 1 N-fastest tile order
template <int BN, int AMN, int BMN, class Epi, int CG = 1, int ST = 0>
static void launch_tc_impl(cudaStream_t st, int M, int N, int K, Mat A, Mat B, const Epi& e, int ks = 1) {
  using C = tc::Cfg<BN, CG, ST>;
  static bool attr = false;
  auto kfn = gemm_tc_kernel<BN, AMN, BMN, Epi, CG, ST>;
  if (!attr) {
    CMT_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  CUtensorMap ta, tb, tcm;
  const void* ap = A.p ? A.p : B.p;
  long long Kx = std::max(K, 64);
  if (AMN) make_map(&ta, ap, M, Kx, A.ld, 64, tc::BK);
  else make_map(&ta, ap, Kx, M, A.ld, tc::BK, tc::BM);
  if (BMN) make_map(&tb, B.p, N, Kx, B.ld, 64, tc::BK);
  else make_map(&tb, B.p, Kx, N, B.ld, tc::BK, C::BNC);
  if constexpr (ST) make_map_c(&tcm, e.C, N, M, e.ldc, e.c_bf16 != 0);
  else tcm = ta;
  int tiles = ceil_div(M, C::TILE_M) * ceil_div(N, BN) * (ks > 0 ? ks : 1);
  const int sms = g_grid_cap > 0 ? std::min(g_num_sms, g_grid_cap) : g_num_sms;
  int grid = ks > 0 ? CG * std::min(tiles, sms / CG) : CG * (sms / CG);
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(grid);
  c.blockDim = dim3(tc::NUM_THREADS);
  c.dynamicSmemBytes = C::SMEM;
  c.stream = st;
  cudaLaunchAttribute at[1];
  int na = 0;
  if (CG > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = CG;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  c.attrs = at;
  c.numAttrs = na;
  CMT_CUDA(cudaLaunchKernelEx(&c, kfn, ta, tb, tcm, M, N, K, e, g_gemm_opt, ks));
  CMT_LAUNCHED(); tl_mark(st, gemm_label(M, N, K, BN, CG));
}

static int g_tma_store = 1;  // option: TMA-store epilogue for EpiStore GEMMs

static int g_splitk = 1;  // option: split-K (TMA reduce-add) for linear fp32 epilogues
// K slices for a linear fp32 EpiStore GEMM whose tile count leaves CTA pairs
// idle in the last wave: minimise waves(tiles * ks) / ks (+ a per-slice cost).
// Returns 1 (no split), 2 (two K slices per tile) or -1 (stream-K).  At most
// two pieces of a tile ever meet in C (zeroed first), and fp32 addition is
// commutative, so the result does not depend on which piece lands first.
static int pick_ks(int M, int N, int K, int BN, int CG) {
  if (!g_splitk) return 1;
  const long long tiles = (long long)ceil_div(M, 128 * CG) * ceil_div(N, BN);
  const long long units = (g_grid_cap > 0 ? std::min(g_num_sms, g_grid_cap) : g_num_sms) / CG;
  const int nkb = ceil_div(K, 64);
  double t1 = (double)((tiles + units - 1) / units);  // in whole-tile times
  int best = 1;
  double best_t = t1;
  if (nkb >= 32) {
    double t2 = (double)((tiles * 2 + units - 1) / units) / 2 + 0.04;
    if (t2 < best_t * 0.95) { best = 2; best_t = t2; }
  }
  // owner/helper stream-K (GemmWork): tiles < units, every tile in two pieces.
  // Off by default (g_splitk & 2): each helper piece pays a full-tile epilogue
  // (TMEM drain + reduce-add), which made the c3 dW GEMMs slower (68 vs 48 us).
  if ((g_splitk & 2) && tiles < units && nkb >= 32) {
    const long long nh = units - tiles, tph = (tiles + nh - 1) / nh;
    double ts = (double)tph / (tph + 1) + 0.04;
    if (ts < best_t * 0.95) { best = -1; best_t = ts; }
  }
  return best;
}

template <int BN, int AMN, int BMN, class Epi, int CG = 1>
static void launch_tc(cudaStream_t st, int M, int N, int K, Mat A, Mat B, const Epi& e) {
  if constexpr (std::is_same<Epi, EpiStore>::value) {
    if (g_tma_store && c_map_ok(e.C, e.ldc, e.c_bf16 != 0) && !(e.beta && e.c_bf16)) {
      int ks = 1;
      // split / stream-K only into a zeroed C (accumulating epilogues would add
      // 2 pieces onto existing values in a timing-dependent order)
      if (!e.c_bf16 && !e.bias && e.act == 0 && !e.add && !e.beta) ks = pick_ks(M, N, K, BN, CG);
      if (ks != 1) {  // pieces reduce-add into a zeroed C
        if (e.ldc == N) CMT_CUDA(cudaMemsetAsync(e.C, 0, (size_t)M * N * 4, st));
        else CMT_CUDA(cudaMemset2DAsync(e.C, (size_t)e.ldc * 4, 0, (size_t)N * 4, M, st));
      }
      return launch_tc_impl<BN, AMN, BMN, Epi, CG, 1>(st, M, N, K, A, B, e, ks);
    }
  }
  launch_tc_impl<BN, AMN, BMN, Epi, CG, 0>(st, M, N, K, A, B, e);
}

// Tile choice for the EpiStore GEMMs: (BN, CG) with the best wave efficiency
// (tiles / (waves * units)); on ties prefer the CTA pair and the wider tile,
// whose per-SM operand stream is smallest.  Encoded as BN * 4 + CG.
static int pick_tile(int M, int N) {
  if (N <= 64) return 64 * 4 + 1;
  // relative per-tile throughput measured with scripts/gemm_bench.py at the c3
  // shapes (256-wide CTA-pair tiles stream the fewest operand bytes per FLOP)
  struct Cand { int bn, cg; double rate; };
  const Cand cands[] = {{256, 2, 1.0}, {128, 2, 0.65}, {256, 1, 0.8}, {128, 1, 0.6}};
  int best = 128 * 4 + 1;
  double best_s = -1;
  for (const Cand& c : cands) {
    if (c.bn > 128 && N <= 128) continue;
    long long units = g_num_sms / c.cg;
    long long t = (long long)ceil_div(M, 128 * c.cg) * ceil_div(N, c.bn);
    long long waves = (t + units - 1) / units;
    double eff = (double)t / (double)(waves * units);
    double s = eff * c.rate;
    if (s > best_s) { best_s = s; best = c.bn * 4 + c.cg; }
  }
  return best;
}

// ---------------------------------------------------------------------------
// Engine
// ---------------------------------------------------------------------------
enum BlockKind { BK_EMB = 0, BK_LSTM_W = 1, BK_LSTM_B = 2, BK_DENSE = 3 };
struct BlockInfo {
  std::string name;
  long long rows, cols;
  int kind;
  int table;      // BK_EMB: 0 src, 1 tgt
  int layer;      // BK_LSTM_*
  int gate;       // 0..3 (i,f,g,o)
  size_t off;     // BK_DENSE: arena offset
};

struct Layer {
  int din;
  size_t w_off, b_off;  // arena offsets: W [din+H][4H], bias [4H]
};

struct Pinned {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t n) {
    if (n > cap) {
      if (p) cudaFreeHost(p);
      CMT_CUDA(cudaMallocHost(&p, n));
      cap = n;
    }
    return p;
  }
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

struct StepOut {  // device -> host step result
  double loss_sum;
  double scal[2];  // sumsq, norm
  int status;
  int pad;
  int flag4[8];  // data parallel: the status word spread one flag per int (combined with ncclMax)
};

class Engine {
 public:
  cmt_config cfg;
  int V, E, H, L;
  bool bf;  // bf16 mode
  int asz;  // activation element size
  cudaStream_t st = nullptr;
  // side stream for independent work of the two scans of a level (their input
  // projections / weight-gradient GEMMs overlap and pack each other's waves)
  cudaStream_t st2 = nullptr;
  // data parallel: gradient buckets are all-reduced on stc as soon as the
  // backward has produced them; the clip waits for stc
  cudaStream_t stc = nullptr;
  cudaEvent_t ev_ar[64] = {};
  int n_ev_ar = 0;
  int ar_overlap = 1;  // option: bucketed all-reduce overlapped with the backward (0: one all-reduce at the end)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // dropout masks generated ahead of their sites on the SMs a scan leaves idle
  struct MaskSite {
    int id;
    uint8_t* keep;
    int N;
    unsigned long long base;
  };
  std::vector<MaskSite> mask_queue;  // generated beside the next recurrent launch
  cudaEvent_t ev_mask[130] = {};
  int mask_ahead = 1;  // option "mask_ahead"
  // background stream: the first columns of a BPTT level's weight grads run
  // here, grid-capped to the SMs the next level's scans leave idle
  cudaStream_t stb = nullptr;
  cudaEvent_t ev_bg = nullptr, ev_bgj = nullptr;
  bool bg_pending = false;
  int bwd_bg = 25;  // option (A/B: 0 9.556, 15 9.531, 25 9.457, 30 9.466, 40 9.68 ms/step at c3): percent of a BPTT level's dW columns computed beside the next scan (0: off)
  std::vector<void*> dUl;  // per-layer dU buffers while the split is on (a deferred GEMM still reads its level's dU)
  int overlap = 1;      // option
  bool on_side = false;
  cudaEvent_t ev[16];
  std::string err;

  std::vector<BlockInfo> blocks;
  std::vector<Layer> layers;  // 0: enc.l1.fwd, 1: enc.l1.bwd, k (2..L): enc.lk, L+k (1..L): dec.lk
  size_t off_wa, off_wc, off_wo, off_bo;
  size_t dense_n = 0;
  float* dw = nullptr;   // dense masters
  float* dg = nullptr;   // dense grads
  bf16* dsh = nullptr;   // dense bf16 shadows
  float* emb_w[2] = {nullptr, nullptr};
  bf16* emb_sh[2] = {nullptr, nullptr};
  int n_tables;

  // workspace
  char* ws = nullptr;
  size_t ws_cap = 0;
  int S = 0, T = 0, B = 0;
  bool staged = false;
  double ntok_local = 0;

  // per-shape carved pointers
  struct LayerWS {
    void* yext;
    float* cext;
    float* acts;
    float* tc;
    float* dy;
  };
  std::vector<LayerWS> lw;
  int *src_ids_d, *tgt_in_d, *tgt_out_d;
  float *src_mask_d, *tgt_mask_d;
  void *Xs, *Xt, *top, *u_att, *cst_att, *hod, *Y, *dhpre, *du_att, *dU, *dU2;
  float* cepart = nullptr;  // per-CTA dY column sums of the fused CE kernel
  float2* cerow = nullptr;  // per-token (lse * log2e, mask / ntok) between the two CE passes
  float* colpart2 = nullptr;  // column-sum scratch of the side stream
  unsigned *colticket = nullptr, *colticket2 = nullptr;  // colsum_partial_v8 tickets (self-resetting)
  float* dho32 = nullptr;   // fp32 split-K scratch of dH_o (bf16 mode)
  float *att_part = nullptr, *att_dsc = nullptr;  // split attention: score slices, d scores
  bf16 *att_a16 = nullptr, *att_d16 = nullptr, *att_dc16 = nullptr;
  int att_tc = 1;  // option: attention core as batched tcgen05 GEMMs (attention_tc.cuh)
  bool att_tc_ok() const { return bf && att_tc && S <= 256 && H % 64 == 0; }
  int s8() const { return (S + 7) / 8 * 8; }
  // one operand of a batched GEMM as a 3-D TMA map (attention_tc.cuh)
  struct BatOp {
    const void* p;
    long long d0, rows;       // contiguous extent, row extent
    long long bstr, rstr;     // batch / row strides in bytes
    int bpos;                 // 1: {d0, batch, rows}, 2: {d0, rows, batch}
  };
  void bat_map(CUtensorMap* m, const BatOp& o, int nb, int box0, int boxr) {
    if (((uintptr_t)o.p & 15) || (o.bstr & 15) || (o.rstr & 15))
      throw Error(CMT_ERR_SHAPE, "batched GEMM operand not 16-byte aligned");
    const bool mid = o.bpos == 1;
    cuuint64_t gdim[3] = {(cuuint64_t)o.d0, (cuuint64_t)(mid ? nb : o.rows), (cuuint64_t)(mid ? o.rows : nb)};
    cuuint64_t gstr[2] = {(cuuint64_t)(mid ? o.bstr : o.rstr), (cuuint64_t)(mid ? o.rstr : o.bstr)};
    cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)(mid ? 1 : boxr), (cuuint32_t)(mid ? boxr : 1)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(o.p), gdim, gstr, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(CMT_ERR_CUDA, "cuTensorMapEncodeTiled (batched) failed: " + std::to_string((int)r));
  }
  // C_b = A_b B_b^T for every batch b (one work unit per (b, tile)); A_MN / B_MN as in gemm.cuh
  template <int BN, int AMN, int BMN>
  void bat_gemm(int M, int N, int K, int nb, const BatOp& A, const BatOp& Bo, const BatStore& e) {
    using C = bat::Cfg<BN>;
    auto kfn = gemm_bat_kernel<BN, AMN, BMN>;
    static bool attr = false;
    if (!attr) {
      CMT_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
      attr = true;
    }
    CUtensorMap ta, tb;
    bat_map(&ta, A, nb, 64, AMN ? 64 : bat::BM);
    bat_map(&tb, Bo, nb, 64, BMN ? 64 : BN);
    const int tiles = nb * ceil_div(M, bat::BM) * ceil_div(N, BN);
    kfn<<<std::min(tiles, g_num_sms), bat::THREADS, C::SMEM, st>>>(ta, tb, M, N, K, nb, A.bpos, Bo.bpos, e);
    CMT_LAUNCHED();
    tl_mark(st, "attn_tc " + gemm_label(M, N, K, BN, 1));
  }
  // scores / dalpha: C_b[T][S] = X_b Hs_b^T with X = U or dC (rows t*B+b, K = H)
  void att_tc_ts(const void* X, float* out) {
    const void* Hs = (L == 1) ? top : views(L, false).ybase;
    const BatOp xa{X, H, T, H * 2LL, (long long)B * H * 2, 1}, hb{Hs, H, S, H * 2LL, (long long)B * H * 2, 1};
    const BatStore e{out, S, (long long)T * S, 0, 0};
    if (S <= 64) bat_gemm<64, 0, 0>(T, S, H, B, xa, hb, e);
    else if (S <= 128) bat_gemm<128, 0, 0>(T, S, H, B, xa, hb, e);
    else bat_gemm<256, 0, 0>(T, S, H, B, xa, hb, e);
  }
  // [T x H] products: C_b = P_b Hs_b with P = alpha or dscores (bf16 [B][T][S8], K = S)
  void att_tc_th(const bf16* P, void* out, long long ldc, long long bstride, int c_bf16) {
    const void* Hs = (L == 1) ? top : views(L, false).ybase;
    const BatOp pa{P, S, T, (long long)T * s8() * 2, s8() * 2LL, 2}, hb{Hs, H, S, H * 2LL, (long long)B * H * 2, 1};
    bat_gemm<256, 0, 1>(T, H, S, B, pa, hb, BatStore{out, ldc, bstride, c_bf16, 0});
  }
  int att_split = 2;  // option: 2 tiled split attention (S,T <= 128), 1 split (<= 64), 0 per-sentence
  int allow_empty_targets = 0;  // option: stage batches with no unmasked target (dev_entropy)
  bool last_infer = false;
  float *ux, *ux2, *ux3, *alpha, *ho, *losstok, *dcst, *dXemb, *dtop, *dhc, *dcc, *colpart;
  std::vector<void*> drop_enc, drop_dec;
  std::vector<uint8_t*> keep_enc, keep_dec;
  uint8_t* keep_o;
  std::vector<float*> fin_dh, fin_dc;
  // embedding compact grads
  int* seg_off_d[2];
  int* seg_pos_d[2];
  int* uniq_d[2];
  float* gcomp[2];
  int nuniq[2] = {0, 0};
  double stage_us[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // host staging phases (debug stat "stage_us:i")
  int nrows_max[2] = {0, 0};  // the most unique rows a batch of the staged shape can have
  // embedding segments built on the device (segments_kernel, in the step) or
  // on the host at staging (data parallel: the ranks exchange their row sets)
  bool seg_dev = false;
  int use_seg_dev = 1;            // option "seg_dev"
  bool seg_host_ok[2] = {false, false};
  std::vector<int> seg_ids_h[2];  // device-segment mode: this batch's ids per table (host copy)
  std::vector<unsigned long long> sort_tmp;  // radix-sort scratch of the segment builder
  int nseg_pos[2] = {0, 0};
  double* normpart;
  unsigned* flags;
  // readiness-flag regions: one per recurrent launch of a step (forward scan of
  // layer l: region l; its BPTT scan: region nlayers + l), sized by the layer
  // count so no two scans of a step ever share counters
  // ParamBlock.learnable (graph.py:20-31): frozen blocks are left out of the
  // global norm and the update (training.py:128-139).  The dense grads enter
  // the norm and the update as segments; in a gate-interleaved LSTM region
  // element i belongs to gate i & 3, so a segment carries a 4-bit gate mask.
  struct GradSeg { size_t off, n; int lanes; };
  std::vector<char> learnable;
  std::vector<GradSeg> segs;
  bool table_learn[2] = {true, true};
  void set_learnable(int idx, bool v) {
    if (idx < 0 || idx >= (int)blocks.size()) throw Error(CMT_ERR_SHAPE, "block index out of range");
    learnable[idx] = v ? 1 : 0;
    rebuild_segs();
  }
  void rebuild_segs() {
    drop_graphs();  // the update's launches depend on the segments
    segs.clear();
    std::vector<int> wm(layers.size(), 0), bm(layers.size(), 0);
    bool all = true;
    for (size_t i = 0; i < blocks.size(); ++i) {
      const BlockInfo& b = blocks[i];
      const bool on = learnable[i] != 0;
      if (b.kind == BK_EMB) { table_learn[b.table] = on; continue; }
      all = all && on;
      if (!on) continue;
      if (b.kind == BK_LSTM_W) wm[b.layer] |= 1 << b.gate;
      else if (b.kind == BK_LSTM_B) bm[b.layer] |= 1 << b.gate;
      else segs.push_back({b.off, (size_t)(b.rows * b.cols), 15});
    }
    if (n_tables == 1) table_learn[1] = table_learn[0];
    if (all) {  // the common case: one segment over the whole arena (alignment gaps are zero)
      segs.assign(1, GradSeg{0, dense_n, 15});
      return;
    }
    for (size_t l = 0; l < layers.size(); ++l) {
      if (wm[l]) segs.push_back({layers[l].w_off, (size_t)(layers[l].din + H) * 4 * H, wm[l]});
      if (bm[l]) segs.push_back({layers[l].b_off, (size_t)4 * H, bm[l]});
    }
  }
  size_t flag_words() const { return 2 * layers.size() * FLAG_STRIDE; }
  unsigned* fwd_flags(int l) const { return flags + (size_t)l * FLAG_STRIDE; }
  unsigned* bwd_flags(int l) const { return flags + (layers.size() + l) * FLAG_STRIDE; }
  int persistent = 1;  // option: persistent recurrent kernels in bf16 mode
  int cg2 = 1;         // option: CTA-pair (cta_group::2) tiles for the large GEMMs
  int dual = 1;        // option: run independent scans of the layer graph two at a time
  int fwd_tm = 1;      // option: forward scans with W_h split over smem + TMEM (lstm_tm.cuh)
  int early_dec1 = 1;  // option: dec.l1's input projection runs beside the enc.l1 scans on the idle SMs
  int ce2 = 2;         // option: fused two-pass CE + bias-grad column sums (0: per-row kernel + column sums)
  bool use_ce2() const { return bf && ce2 && V % 8 == 0; }
  // data parallel (NCCL): dense all-reduce of grads, loss and status
  void* comm = nullptr;
  int rank = 0, world = 1;
  // data parallel: the embedding grads are exchanged as rows of the UNION of all
  // ranks' touched ids (cmt_set_union, computed by the host from every rank's
  // staged ids): ubuf[t] [U][E] holds this rank's rows at their union index
  // (zeros elsewhere) and is all-reduced; the norm and the update then run
  // over the U union rows on every rank (identical results everywhere).
  float* ubuf[2] = {nullptr, nullptr};
  int *umap_d[2] = {nullptr, nullptr}, *uids_d[2] = {nullptr, nullptr};
  size_t ucap[2] = {0, 0};
  int nunion[2] = {0, 0};
  bool union_set[2] = {false, false};
  bool emb_sent[2] = {false, false};
  void set_union(int t, const int* ids, int n) {
    if (t < 0 || t >= n_tables) throw Error(CMT_ERR_SHAPE, "table index out of range");
    if (!staged) throw Error(CMT_ERR_CONFIG, "stage the batch before setting its rows union");
    host_segments(t);
    std::vector<int> map((size_t)nuniq[t]);
    int j = 0;
    for (int i = 0; i < n; ++i) {
      if (ids[i] < 0 || ids[i] >= V || (i && ids[i] <= ids[i - 1]))
        throw Error(CMT_ERR_CONFIG, "rows union must be ascending unique ids in [0, V)");
      if (j < nuniq[t] && uniq_h[t][j] == ids[i]) map[j++] = i;
    }
    if (j != nuniq[t]) throw Error(CMT_ERR_CONFIG, "rows union does not contain this rank's ids");
    if ((size_t)n > ucap[t]) {
      for (void* q : {(void*)ubuf[t], (void*)umap_d[t], (void*)uids_d[t]}) if (q) CMT_CUDA(cudaFree(q));
      CMT_CUDA(cudaMalloc(&ubuf[t], (size_t)n * E * 4));
      CMT_CUDA(cudaMalloc(&umap_d[t], (size_t)std::max(n, 1) * 4));  // >= this rank's rows
      CMT_CUDA(cudaMalloc(&uids_d[t], (size_t)n * 4));
      ucap[t] = n;
    }
    CMT_CUDA(cudaStreamSynchronize(st));
    if (nuniq[t]) CMT_CUDA(cudaMemcpy(umap_d[t], map.data(), map.size() * 4, cudaMemcpyHostToDevice));
    if (n) CMT_CUDA(cudaMemcpy(uids_d[t], ids, (size_t)n * 4, cudaMemcpyHostToDevice));
    nunion[t] = n;
    union_set[t] = true;
  }

  void nccl_check(int r, const char* what) {
    if (r != 0)
      throw Error(CMT_ERR_CUDA, std::string(what) + ": " + (g_nccl.get_error ? g_nccl.get_error(r) : "nccl error"));
  }
  void set_comm(const void* uid, int rank_, int world_) {
    if (world_ < 1 || rank_ < 0 || rank_ >= world_) throw Error(CMT_ERR_CONFIG, "bad rank/world");
    if (comm) throw Error(CMT_ERR_CONFIG, "communicator already set");
    drop_graphs();
    g_nccl.load();
    typedef int (*InitFn)(void**, int, NcclUid, int);
    InitFn init = (InitFn)dlsym(g_nccl.h, "ncclCommInitRank");
    if (!init) throw Error(CMT_ERR_CUDA, "ncclCommInitRank missing");
    NcclUid u;
    std::memcpy(u.internal, uid, 128);
    nccl_check(init(&comm, world_, u, rank_), "ncclCommInitRank");
    rank = rank_;
    world = world_;
    CMT_CUDA(cudaStreamCreateWithFlags(&stc, cudaStreamNonBlocking));
    for (auto& e : ev_ar) CMT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // all-reduce (sum) of a finished gradient bucket on the comm stream, ordered
  // after the work issued so far on the current stream.  Every rank issues the
  // same buckets in the same (host program) order.
  bool ar_buckets = false;    // this step all-reduces gradient buckets during the backward
  std::vector<char> ar_done;  // per bucket: layers 0..2L, attention 2L+1, output 2L+2
  void allreduce_region(int id) {
    if (!ar_buckets || ar_done[id]) return;
    ar_done[id] = 1;
    if (id < (int)layers.size()) {
      const Layer& ly = layers[id];
      allreduce_bucket(dg + ly.w_off, ly.b_off + 4 * (size_t)H - ly.w_off);  // [W; b] of the layer
    } else if (id == (int)layers.size()) {
      allreduce_bucket(dg + off_wa, off_wo - off_wa);  // att.w_a, att.w_c
    } else {
      allreduce_bucket(dg + off_wo, dense_n - off_wo);  // out.w, out.b
    }
  }
  void allreduce_bucket(void* buf, size_t n, int dtype = NCCL_FLOAT32, int op = NCCL_SUM) {
    const int slot = n_ev_ar < 63 ? n_ev_ar++ : 63;  // events are reusable once waited on
    CMT_CUDA(cudaEventRecord(ev_ar[slot], st));
    CMT_CUDA(cudaStreamWaitEvent(stc, ev_ar[slot], 0));
    nccl_check(g_nccl.all_reduce(buf, buf, n, dtype, op, comm, stc), "ncclAllReduce");
  }
  void allreduce_join() {
    if (!n_ev_ar) return;
    CMT_CUDA(cudaEventRecord(ev_ar[0], stc));
    CMT_CUDA(cudaStreamWaitEvent(st, ev_ar[0], 0));
    n_ev_ar = 0;
  }
  // Every collective of a step is issued on ONE stream (stc while buckets are
  // in flight, else the engine stream), so all ranks execute the shared
  // communicator's operations in the same order.
  void allreduce(void* buf, size_t n, int dtype, int op = NCCL_SUM) {
    if (ar_buckets) {
      allreduce_bucket(buf, n, dtype, op);
      return;
    }
    nccl_check(g_nccl.all_reduce(buf, buf, n, dtype, op, comm, st), "ncclAllReduce");
  }
  int trace_layer = -1;  // debug: record per-step phase timestamps of this layer's forward scan
  unsigned long long* trace_d = nullptr;
  StepScalars* scal_d;
  StepOut* out_d;
  float* s32_d;
  int* status_d;
  double* losssum_d;
  double* normscal_d;
  Pinned pin_in[2], pin_out;  // batch staging is double-buffered (see stage())
  cudaEvent_t pin_ev[2] = {nullptr, nullptr};
  int pin_cur = 0;
  StepOut* out_h = nullptr;
  // host copies of the staged segment info (for grad download)
  std::vector<int> uniq_h[2];

  Engine(const cmt_config& c, int device) : cfg(c) {
    CMT_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    CMT_CUDA(cudaGetDeviceProperties(&prop, device));
    g_num_sms = prop.multiProcessorCount;
    V = c.vocab_size; E = c.embedding_size; H = c.hidden_size; L = c.depth;
    if (V < 1 || E < 1 || H < 1 || L < 1) throw Error(CMT_ERR_CONFIG, "model dims must be positive");
    if (!(c.dropout >= 0.0 && c.dropout < 1.0)) throw Error(CMT_ERR_CONFIG, "dropout must be in [0, 1)");
    bf = c.mode == CMT_MODE_BF16;
    if (bf && prop.major < 10) throw Error(CMT_ERR_CUDA, "bf16 tcgen05 mode needs an sm_100 GPU");
    if (bf && ((E % 8) || (H % 8) || (V % 8)))
      throw Error(CMT_ERR_SHAPE, "bf16 mode needs vocab/embedding/hidden sizes that are multiples of 8");
    asz = bf ? 2 : 4;
    CMT_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CMT_CUDA(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
    CMT_CUDA(cudaStreamCreateWithFlags(&stb, cudaStreamNonBlocking));
    CMT_CUDA(cudaEventCreateWithFlags(&ev_bg, cudaEventDisableTiming));
    CMT_CUDA(cudaEventCreateWithFlags(&ev_bgj, cudaEventDisableTiming));
    CMT_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    CMT_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    for (auto& e : ev_mask) CMT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : pin_ev) CMT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : ev) CMT_CUDA(cudaEventCreate(&e));
    build_registry();
    learnable.assign(blocks.size(), 1);
    rebuild_segs();
    alloc_params();
    out_h = (StepOut*)pin_out.get(sizeof(StepOut));
  }
  ~Engine() {
    cudaStreamSynchronize(st);
    drop_graphs();
    for (cudaEvent_t ev : ev_pool) cudaEventDestroy(ev);
    for (auto& v : probe_ev)
      for (auto& pr : v) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    cudaFree(dw); cudaFree(dg); cudaFree(dsh); cudaFree(gate_stage_d);
    for (int i = 0; i < 2; ++i) {
      if (i == 0 || !cfg.shared_embeddings) { cudaFree(emb_w[i]); cudaFree(emb_sh[i]); }
    }
    cudaFree(ws);
    for (auto& sn : snaps) {
      if (sn.dense) cudaFree(sn.dense);
      for (int t = 0; t < n_tables; ++t)
        if (sn.emb[t]) cudaFree(sn.emb[t]);
    }
    beam_free();
    if (jump_d) cudaFree(jump_d);
    for (int t = 0; t < 2; ++t)
      for (void* q : {(void*)ubuf[t], (void*)umap_d[t], (void*)uids_d[t]}) if (q) cudaFree(q);
    if (comm && g_nccl.comm_destroy) g_nccl.comm_destroy(comm);
    if (stc) {
      cudaStreamDestroy(stc);
      for (auto& e : ev_ar) cudaEventDestroy(e);
    }
    for (auto& e : ev) cudaEventDestroy(e);
    cudaStreamDestroy(st);
    cudaStreamDestroy(st2);
    cudaStreamDestroy(stb);
    cudaEventDestroy(ev_bg);
    cudaEventDestroy(ev_bgj);
    cudaEventDestroy(ev_fork);
    cudaEventDestroy(ev_join);
    for (auto& e : pin_ev) cudaEventDestroy(e);
  }

  static size_t al(size_t x) { return (x + 63) & ~(size_t)63; }

  // Host<->device copies are ordered on the engine stream: a plain cudaMemcpy
  // from pageable memory may return before its DMA lands, racing kernels that
  // run on this non-blocking stream (e.g. the bf16 shadow refresh).
  void copy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    CMT_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, st));
    CMT_CUDA(cudaStreamSynchronize(st));
  }

  void build_registry() {
    n_tables = cfg.shared_embeddings ? 1 : 2;
    blocks.push_back({"src_embed", V, E, BK_EMB, 0, -1, -1, 0});
    if (!cfg.shared_embeddings) blocks.push_back({"tgt_embed", V, E, BK_EMB, 1, -1, -1, 0});
    size_t off = 0;
    auto add_layer = [&](const std::string& prefix, int din) {
      Layer ly;
      ly.din = din;
      ly.w_off = off; off = al(off + (size_t)(din + H) * 4 * H);
      ly.b_off = off; off = al(off + (size_t)4 * H);
      int li = (int)layers.size();
      layers.push_back(ly);
      const char* g = "ifgo";
      for (int q = 0; q < 4; ++q)
        blocks.push_back({prefix + ".w_" + g[q], din + H, H, BK_LSTM_W, -1, li, q, 0});
      for (int q = 0; q < 4; ++q) blocks.push_back({prefix + ".b_" + g[q], H, 1, BK_LSTM_B, -1, li, q, 0});
    };
    add_layer("enc.l1.fwd", E);
    add_layer("enc.l1.bwd", E);
    for (int k = 2; k <= L; ++k) add_layer("enc.l" + std::to_string(k), H);
    for (int k = 1; k <= L; ++k) add_layer("dec.l" + std::to_string(k), k == 1 ? E : H);
    off_wa = off; off = al(off + (size_t)H * H);
    off_wc = off; off = al(off + (size_t)2 * H * H);
    off_wo = off; off = al(off + (size_t)H * V);
    off_bo = off; off = al(off + (size_t)V);
    dense_n = off;
    blocks.push_back({"att.w_a.w", H, H, BK_DENSE, -1, -1, -1, off_wa});
    blocks.push_back({"att.w_c.w", 2LL * H, H, BK_DENSE, -1, -1, -1, off_wc});
    blocks.push_back({"out.w", H, V, BK_DENSE, -1, -1, -1, off_wo});
    blocks.push_back({"out.b", V, 1, BK_DENSE, -1, -1, -1, off_bo});
  }

  void alloc_params() {
    CMT_CUDA(cudaMalloc(&dw, dense_n * 4));
    CMT_CUDA(cudaMalloc(&dg, dense_n * 4));
    CMT_CUDA(cudaMemset(dw, 0, dense_n * 4));
    CMT_CUDA(cudaMemset(dg, 0, dense_n * 4));
    if (bf) {
      CMT_CUDA(cudaMalloc(&dsh, dense_n * 2));
      CMT_CUDA(cudaMemset(dsh, 0, dense_n * 2));
    }
    for (int i = 0; i < n_tables; ++i) {
      CMT_CUDA(cudaMalloc(&emb_w[i], (size_t)V * E * 4));
      CMT_CUDA(cudaMemset(emb_w[i], 0, (size_t)V * E * 4));
      if (bf) CMT_CUDA(cudaMalloc(&emb_sh[i], (size_t)V * E * 2));
    }
    if (n_tables == 1) { emb_w[1] = emb_w[0]; emb_sh[1] = emb_sh[0]; }
  }

  // ---- weight views used by the GEMMs (bf16 shadow or fp32 master) ----
  const void* wv(size_t off) const { return bf ? (const void*)(dsh + off) : (const void*)(dw + off); }
  const void* table_v(int t) const { return bf ? (const void*)emb_sh[t] : (const void*)emb_w[t]; }
  int tgt_table() const { return cfg.shared_embeddings ? 0 : 1; }

  // ---- upload / download ----
  void check_block(int idx, long long rows, long long cols) {
    if (idx < 0 || idx >= (int)blocks.size()) throw Error(CMT_ERR_SHAPE, "block index out of range");
    if (blocks[idx].rows != rows || blocks[idx].cols != cols)
      throw Error(CMT_ERR_SHAPE, "shape mismatch for " + blocks[idx].name);
  }
  void upload(int idx, const float* h, long long rows, long long cols) {
    check_block(idx, rows, cols);
    const BlockInfo& b = blocks[idx];
    CMT_CUDA(cudaStreamSynchronize(st));
    if (b.kind == BK_EMB) {
      copy_sync(emb_w[b.table], h, (size_t)rows * cols * 4, cudaMemcpyHostToDevice);
      if (bf) refresh_shadow(emb_w[b.table], emb_sh[b.table], (size_t)rows * cols);
      return;
    }
    if (b.kind == BK_DENSE) {
      copy_sync(dw + b.off, h, (size_t)rows * cols * 4, cudaMemcpyHostToDevice);
      if (bf) refresh_shadow(dw + b.off, dsh + b.off, (size_t)rows * cols);
      return;
    }
    // LSTM gate block: H2D of exactly this block, interleaved on the device
    const Layer& ly = layers[b.layer];
    const size_t n = (size_t)rows * cols;
    float* stage_d = gate_stage(n);
    copy_sync(stage_d, h, n * 4, cudaMemcpyHostToDevice);
    const size_t off = b.kind == BK_LSTM_W ? ly.w_off : ly.b_off;
    const long long grows = b.kind == BK_LSTM_W ? rows : 1;  // a bias is one row of H
    gate_copy_kernel<<<grid_for((long long)n), 256, 0, st>>>(dw + off, stage_d, grows, H, b.gate, 1);
    CMT_LAUNCHED(); tl_mark(st, "gate_copy_kernel");
    if (bf) refresh_shadow(dw + off, dsh + off, (size_t)grows * 4 * H);
    else CMT_CUDA(cudaStreamSynchronize(st));
  }
  float* gate_stage_d = nullptr;  // staging of one LSTM gate block for upload / download
  size_t gate_stage_n = 0;
  float* gate_stage(size_t n) {
    if (n > gate_stage_n) {
      if (gate_stage_d) CMT_CUDA(cudaFree(gate_stage_d));
      CMT_CUDA(cudaMalloc(&gate_stage_d, n * 4));
      gate_stage_n = n;
    }
    return gate_stage_d;
  }
  void refresh_shadow(const float* s, bf16* d, size_t n) {
    to_bf16_kernel<<<std::min<long long>(4096, ceil_div(n, 256)), 256, 0, st>>>(s, d, (long long)n);
    CMT_LAUNCHED(); tl_mark(st, "to_bf16_kernel");
    CMT_CUDA(cudaStreamSynchronize(st));
  }
  void download(int idx, float* h, long long rows, long long cols, bool grad, int snap = -1) {
    check_block(idx, rows, cols);
    CMT_CUDA(cudaStreamSynchronize(st));
    const BlockInfo& b = blocks[idx];
    if (snap >= 0 && !snaps[snap].dense) throw Error(CMT_ERR_CONFIG, "snapshot slot is empty");
    const float* base = snap >= 0 ? snaps[snap].dense : grad ? dg : dw;
    if (b.kind == BK_EMB) {
      if (!grad) {
        copy_sync(h, snap >= 0 ? snaps[snap].emb[b.table] : emb_w[b.table], (size_t)rows * cols * 4,
                  cudaMemcpyDeviceToHost);
      } else {
        std::memset(h, 0, (size_t)rows * cols * 4);
        int t = b.table;
        int n = host_rows(t);
        if (n > 0) {
          std::vector<float> gc((size_t)n * E);
          copy_sync(gc.data(), gcomp[t], gc.size() * 4, cudaMemcpyDeviceToHost);
          for (int u = 0; u < n; ++u) std::memcpy(h + (size_t)uniq_h[t][u] * E, &gc[(size_t)u * E], E * 4);
        }
      }
      return;
    }
    if (b.kind == BK_DENSE) {
      copy_sync(h, base + b.off, (size_t)rows * cols * 4, cudaMemcpyDeviceToHost);
      return;
    }
    // LSTM gate block: de-interleaved on the device, D2H of exactly this block
    const Layer& ly = layers[b.layer];
    const size_t n = (size_t)rows * cols;
    float* stage_d = gate_stage(n);
    const size_t off = b.kind == BK_LSTM_W ? ly.w_off : ly.b_off;
    const long long grows = b.kind == BK_LSTM_W ? rows : 1;  // a bias is one row of H
    gate_copy_kernel<<<grid_for((long long)n), 256, 0, st>>>(const_cast<float*>(base) + off, stage_d, grows, H,
                                                            b.gate, 0);
    CMT_LAUNCHED(); tl_mark(st, "gate_copy_kernel");
    copy_sync(h, stage_d, n * 4, cudaMemcpyDeviceToHost);
  }

  // ---- device-resident parameter snapshots (ModelParams.copy_data/load_data,
  // model.py:104-115; the Trainer's restore-from-best, training.py:246-254):
  // fp32 masters copied device-to-device, no host round trip ----
  struct Snapshot {
    float* dense = nullptr;
    float* emb[2] = {nullptr, nullptr};
  };
  static constexpr int NSNAP = 4;
  Snapshot snaps[NSNAP];
  void check_slot(int slot) const {
    if (slot < 0 || slot >= NSNAP) throw Error(CMT_ERR_CONFIG, "snapshot slot out of range");
  }
  void snapshot_save(int slot) {
    check_slot(slot);
    Snapshot& sn = snaps[slot];
    if (!sn.dense) {
      CMT_CUDA(cudaMalloc(&sn.dense, dense_n * 4));
      for (int t = 0; t < n_tables; ++t) CMT_CUDA(cudaMalloc(&sn.emb[t], (size_t)V * E * 4));
    }
    CMT_CUDA(cudaMemcpyAsync(sn.dense, dw, dense_n * 4, cudaMemcpyDeviceToDevice, st));
    for (int t = 0; t < n_tables; ++t)
      CMT_CUDA(cudaMemcpyAsync(sn.emb[t], emb_w[t], (size_t)V * E * 4, cudaMemcpyDeviceToDevice, st));
    CMT_CUDA(cudaStreamSynchronize(st));
  }
  void snapshot_restore(int slot) {
    check_slot(slot);
    const Snapshot& sn = snaps[slot];
    if (!sn.dense) throw Error(CMT_ERR_CONFIG, "snapshot slot is empty");
    CMT_CUDA(cudaMemcpyAsync(dw, sn.dense, dense_n * 4, cudaMemcpyDeviceToDevice, st));
    for (int t = 0; t < n_tables; ++t)
      CMT_CUDA(cudaMemcpyAsync(emb_w[t], sn.emb[t], (size_t)V * E * 4, cudaMemcpyDeviceToDevice, st));
    if (bf) {
      refresh_shadow(dw, dsh, dense_n);
      for (int t = 0; t < n_tables; ++t) refresh_shadow(emb_w[t], emb_sh[t], (size_t)V * E);
    }
    CMT_CUDA(cudaStreamSynchronize(st));
  }
  void snapshot_free(int slot) {
    check_slot(slot);
    Snapshot& sn = snaps[slot];
    CMT_CUDA(cudaStreamSynchronize(st));
    if (sn.dense) cudaFree(sn.dense);
    for (int t = 0; t < n_tables; ++t)
      if (sn.emb[t]) cudaFree(sn.emb[t]);
    sn = Snapshot();
  }

  // ---- batched beam search on the device (decode.cuh):
  // every live hypothesis of every sentence of a batch is a row of one decoder
  // step (model.py:211-236); the beam bookkeeping of decoding.py:89-153 runs
  // in beam_select_kernel.  The encoder is the training forward in INFER mode
  // on the padded batch (padding carries state / is masked out exactly, so a
  // sentence's states equal those of encoding it alone). ----
  struct BeamWs {
    int B = 0, K = 0, kk = 0, nb = 0, S = 0, Tmax = 0, rows = 0, cur = 0;
    bool ready = false, finished = false;
    char* mem = nullptr;
    size_t cap = 0;
    void* hs = nullptr;
    float *smask, *fin_h, *fin_c, *hst[2], *cst[2], *cin, *U, *u, *Y, *topv;
    void *zc, *ho;
    void* z[64];
    void** zp_d;
    int *zld_d, *zoff_d, *topi, *ids, *par, *nactive;
    BeamSent* sent;
    double *live_lp, *lptab;
    int2* bp;
    BeamFin* fin;
    std::vector<BeamSent> h_sent;
    std::vector<BeamFin> h_fin;
    std::vector<int2> h_bp;
    std::vector<double> h_lp;
  } bw;
  int* bw_active_h = nullptr;  // pinned
  void beam_free() {
    if (bw.mem) cudaFree(bw.mem);
    bw.mem = nullptr;
    bw.cap = 0;
    if (bw_active_h) cudaFreeHost(bw_active_h);
    bw_active_h = nullptr;
  }
  void beam_begin(const long long* src, const float* smask, int S_, int B_, int beam, int n_best, const int* max_len,
                  const double* lptab, int nlp) {
    if (S_ < 1 || B_ < 1) throw Error(CMT_ERR_SHAPE, "beam search needs a (S >= 1, B >= 1) source batch");
    if (beam < 1 || beam > bm::MAXK) throw Error(CMT_ERR_CONFIG, "beam_size must be in [1, 32]");
    if (L > 63) throw Error(CMT_ERR_CONFIG, "beam search supports depth <= 63");
    int Tmax = 0;
    for (int b = 0; b < B_; ++b) {
      if (max_len[b] < 1) throw Error(CMT_ERR_CONFIG, "max_len must be >= 1");
      Tmax = std::max(Tmax, max_len[b]);
    }
    if (nlp < Tmax + 2) throw Error(CMT_ERR_SHAPE, "length-penalty table shorter than max_len + 2");
    // encoder: the training forward in INFER mode on the padded batch (dummy target row)
    std::vector<long long> eos((size_t)B_, 3);
    std::vector<float> one((size_t)B_, 1.f);
    stage(src, smask, S_, eos.data(), one.data(), 1, B_);
    cmt_step_args a = {};
    a.flags = CMT_FLAG_INFER;
    a.pcg_inc_lo = 1;
    cmt_step_result r = {};
    run(a, &r);
    if (r.status != CMT_OK) throw Error(r.status, "non-finite values while encoding the source");
    BeamWs& w = bw;
    w.B = B_; w.K = beam; w.kk = std::min(beam, V); w.nb = std::max(n_best, 1); w.S = S_; w.Tmax = Tmax;
    w.rows = B_ * beam; w.cur = 0; w.finished = false;
    const long long rows = w.rows, SB = (long long)S_ * B_;
    const int zc = std::max(E, H) + H;
    // carve one allocation
    size_t need = 0;
    auto sz = [&](size_t bytes) { size_t o = need; need += (bytes + 255) & ~(size_t)255; return o; };
    const size_t o_hs = sz(SB * H * asz), o_sm = sz(SB * 4), o_fh = sz((size_t)L * B_ * H * 4),
                 o_fc = sz((size_t)L * B_ * H * 4);
    size_t o_h[2], o_c[2];
    for (int q = 0; q < 2; ++q) { o_h[q] = sz((size_t)L * rows * H * 4); o_c[q] = sz((size_t)L * rows * H * 4); }
    const size_t o_cin = sz((size_t)L * rows * H * 4), o_U = sz((size_t)rows * 4 * H * 4), o_u = sz((size_t)rows * H * 4),
                 o_Y = sz((size_t)rows * V * 4), o_tv = sz((size_t)rows * w.kk * 4), o_ti = sz((size_t)rows * w.kk * 4),
                 o_zc = sz((size_t)rows * 2 * H * asz), o_ho = sz((size_t)rows * H * asz);
    size_t o_z[64];
    for (int k = 0; k < L; ++k) o_z[k] = sz((size_t)rows * zc * asz);
    const size_t o_zp = sz(64 * sizeof(void*)), o_zld = sz(64 * 4), o_zoff = sz(64 * 4), o_ids = sz(rows * 4),
                 o_par = sz(rows * 4), o_na = sz(4), o_sent = sz((size_t)B_ * sizeof(BeamSent)),
                 o_llp = sz((size_t)rows * 8), o_lpt = sz((size_t)nlp * 8),
                 o_bp = sz((size_t)B_ * Tmax * beam * sizeof(int2)), o_fin = sz((size_t)B_ * w.nb * sizeof(BeamFin));
    if (need > w.cap) {
      if (w.mem) CMT_CUDA(cudaFree(w.mem));
      CMT_CUDA(cudaMalloc(&w.mem, need));
      w.cap = need;
    }
    if (!bw_active_h) CMT_CUDA(cudaMallocHost(&bw_active_h, 4));
    char* m0 = w.mem;
    w.hs = m0 + o_hs; w.smask = (float*)(m0 + o_sm); w.fin_h = (float*)(m0 + o_fh); w.fin_c = (float*)(m0 + o_fc);
    for (int q = 0; q < 2; ++q) { w.hst[q] = (float*)(m0 + o_h[q]); w.cst[q] = (float*)(m0 + o_c[q]); }
    w.cin = (float*)(m0 + o_cin); w.U = (float*)(m0 + o_U); w.u = (float*)(m0 + o_u); w.Y = (float*)(m0 + o_Y);
    w.topv = (float*)(m0 + o_tv); w.topi = (int*)(m0 + o_ti); w.zc = m0 + o_zc; w.ho = m0 + o_ho;
    for (int k = 0; k < L; ++k) w.z[k] = m0 + o_z[k];
    w.zp_d = (void**)(m0 + o_zp); w.zld_d = (int*)(m0 + o_zld); w.zoff_d = (int*)(m0 + o_zoff);
    w.ids = (int*)(m0 + o_ids); w.par = (int*)(m0 + o_par); w.nactive = (int*)(m0 + o_na);
    w.sent = (BeamSent*)(m0 + o_sent); w.live_lp = (double*)(m0 + o_llp); w.lptab = (double*)(m0 + o_lpt);
    w.bp = (int2*)(m0 + o_bp); w.fin = (BeamFin*)(m0 + o_fin);
    // encoder outputs: the top layer (rows s*B + b), the mask, the finals (model.py:207-208)
    const void* Hs = (L == 1) ? top : views(L, false).ybase;
    CMT_CUDA(cudaMemcpyAsync(w.hs, Hs, SB * H * asz, cudaMemcpyDeviceToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(w.smask, src_mask_d, SB * 4, cudaMemcpyDeviceToDevice, st));
    const long long BH = (long long)B_ * H;
    for (int k = 1; k <= L; ++k) {  // l1.bwd's final sits in slot 0, deep layers' in slot S
      const int el = (k == 1) ? 1 : k;
      const size_t slot = (k == 1) ? 0 : (size_t)S_;
      const void* hsrc = (const char*)lw[el].yext + slot * BH * asz;
      if (bf) copy2d_kernel<bf16, float><<<grid_for(BH), 256, 0, st>>>((const bf16*)hsrc, BH, w.fin_h + (k - 1) * BH, BH, 1, (int)BH);
      else copy2d_kernel<float, float><<<grid_for(BH), 256, 0, st>>>((const float*)hsrc, BH, w.fin_h + (k - 1) * BH, BH, 1, (int)BH);
      CMT_LAUNCHED(); tl_mark(st, "copy2d_kernel");
      CMT_CUDA(cudaMemcpyAsync(w.fin_c + (k - 1) * BH, lw[el].cext + slot * BH, BH * 4, cudaMemcpyDeviceToDevice, st));
    }
    // layer inputs z_k = [x | h_prev]: x is E (k = 1) or H wide
    std::vector<void*> zp(64, nullptr);
    std::vector<int> zld(64, 0), zoff(64, 0);
    for (int k = 0; k < L; ++k) {
      const int din = layers[L + 1 + k].din;
      zp[k] = w.z[k]; zld[k] = din + H; zoff[k] = din;
    }
    CMT_CUDA(cudaMemcpyAsync(w.zp_d, zp.data(), 64 * sizeof(void*), cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(w.zld_d, zld.data(), 64 * 4, cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(w.zoff_d, zoff.data(), 64 * 4, cudaMemcpyHostToDevice, st));
    // beam state: one live hypothesis (no tokens, log-prob 0) per sentence, fed BOS
    std::vector<BeamSent> sent((size_t)B_);
    for (int b = 0; b < B_; ++b) {
      BeamSent& q = sent[b];
      q = BeamSent{};
      q.n_live = 1; q.max_len = max_len[b]; q.trunc_slot = -1;
      q.best_fin = -INFINITY; q.lp_cap = lptab[max_len[b]];
    }
    std::vector<int> ids((size_t)rows, 2), par((size_t)rows, -1);
    std::vector<double> llp((size_t)rows, 0.0);
    CMT_CUDA(cudaMemcpyAsync(w.sent, sent.data(), sent.size() * sizeof(BeamSent), cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(w.ids, ids.data(), rows * 4, cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(w.par, par.data(), rows * 4, cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(w.live_lp, llp.data(), rows * 8, cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(w.lptab, lptab, (size_t)nlp * 8, cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaStreamSynchronize(st));
    w.ready = true;
  }
  template <typename A>
  void beam_step_t() {
    BeamWs& w = bw;
    const int rows = w.rows, in = w.cur, out = w.cur ^ 1;
    const long long RH = (long long)rows * H;
    beam_gather_kernel<A><<<dim3(rows, L), 256, 0, st>>>(w.hst[in], w.cst[in], w.fin_h, w.fin_c, w.par, rows, w.K,
                                                          w.B, H, (A* const*)w.zp_d, w.zld_d, w.zoff_d, w.cin);
    CMT_LAUNCHED(); tl_mark(st, "beam_gather_kernel");
    beam_embed_kernel<A><<<rows, 128, 0, st>>>((const A*)table_v(tgt_table()), w.ids, E, (A*)w.z[0],
                                                layers[L + 1].din + H);
    CMT_LAUNCHED(); tl_mark(st, "beam_embed_kernel");
    for (int k = 1; k <= L; ++k) {  // decoder layers (lstm_cell_forward, layers.py:344-363)
      const Layer& ly = layers[L + k];
      EpiStore e = store(w.U, 4LL * H, false);
      e.bias = dw + ly.b_off;
      gemm(rows, 4 * H, ly.din + H, Mat{w.z[k - 1], ly.din + H, 0}, Mat{wv(ly.w_off), 4LL * H, 1}, e);
      A* xn = (k < L) ? (A*)w.z[k] : (A*)w.zc + H;  // next layer's x, or h_top into [ctx | h_top]
      const int ldx = (k < L) ? layers[L + k + 1].din + H : 2 * H;
      beam_cell_kernel<A><<<dim3(rows, ceil_div(H, 256)), 256, 0, st>>>(w.U, w.cin + (k - 1) * RH, H,
                                                                         w.hst[out] + (k - 1) * RH,
                                                                         w.cst[out] + (k - 1) * RH, xn, ldx);
      CMT_LAUNCHED(); tl_mark(st, "beam_cell_kernel");
    }
    // attention (attend_values, attention.py:235-250): u = W_a^T h_top, context, H_o = tanh(W_c^T [ctx; h_top])
    gemm(rows, H, H, Mat{(A*)w.zc + H, 2LL * H, 0}, Mat{wv(off_wa), H, 1}, store(w.u, H, false));
    beam_attention_kernel<A><<<rows, bm::ATT_THREADS, (size_t)w.S * 4, st>>>((const A*)w.hs, w.S, w.B, H, w.smask,
                                                                              w.u, w.K, (A*)w.zc, 2 * H);
    CMT_LAUNCHED(); tl_mark(st, "beam_attention_kernel");
    {
      EpiStore e = store(w.ho, H, true);
      e.act = 1;
      gemm(rows, H, 2 * H, Mat{w.zc, 2LL * H, 0}, Mat{wv(off_wc), H, 1}, e);
    }
    {  // output layer (model.py:232-235), fp32 logits
      EpiStore e = store(w.Y, V, false);
      e.bias = dw + off_bo;
      e.act = cfg.output_tanh ? 1 : 0;
      gemm(rows, V, H, Mat{w.ho, H, 0}, Mat{wv(off_wo), V, 1}, e);
    }
    CMT_CUDA(cudaMemsetAsync(w.nactive, 0, 4, st));
    beam_topk_kernel<<<rows, bm::TOPK_THREADS, 0, st>>>(w.Y, V, w.kk, w.K, w.sent, w.topv, w.topi, status_d);
    CMT_LAUNCHED(); tl_mark(st, "beam_topk_kernel");
    beam_select_kernel<<<w.B, 32, 0, st>>>(w.sent, w.live_lp, w.topv, w.topi, w.K, w.kk, w.K, w.bp, w.Tmax, w.fin,
                                           w.nb, w.lptab, w.ids, w.par, w.nactive, 3);
    CMT_LAUNCHED(); tl_mark(st, "beam_select_kernel");
    w.cur = out;
  }
  int beam_step(int max_steps) {
    if (!bw.ready) throw Error(CMT_ERR_CONFIG, "beam_step before beam_begin");
    int active = bw.finished ? 0 : 1;
    CMT_CUDA(cudaMemsetAsync(status_d, 0, 4, st));
    for (int i = 0; i < max_steps && active; ++i) {
      if (bf) beam_step_t<bf16>();
      else beam_step_t<float>();
      CMT_CUDA(cudaMemcpyAsync(bw_active_h, bw.nactive, 4, cudaMemcpyDeviceToHost, st));
      CMT_CUDA(cudaStreamSynchronize(st));
      active = *bw_active_h;
      int stt = 0;
      CMT_CUDA(cudaMemcpy(&stt, status_d, 4, cudaMemcpyDeviceToHost));
      if (stt & ST_LOGITS) throw Error(CMT_ERR_NUM_LOGITS, "log_softmax_columns received non-finite input");
    }
    if (!active && !bw.finished) {  // read the search results back once
      BeamWs& w = bw;
      w.h_sent.resize(w.B);
      w.h_fin.resize((size_t)w.B * w.nb);
      w.h_bp.resize((size_t)w.B * w.Tmax * w.K);
      w.h_lp.resize((size_t)w.rows);
      copy_sync(w.h_sent.data(), w.sent, w.h_sent.size() * sizeof(BeamSent), cudaMemcpyDeviceToHost);
      copy_sync(w.h_fin.data(), w.fin, w.h_fin.size() * sizeof(BeamFin), cudaMemcpyDeviceToHost);
      copy_sync(w.h_bp.data(), w.bp, w.h_bp.size() * sizeof(int2), cudaMemcpyDeviceToHost);
      copy_sync(w.h_lp.data(), w.live_lp, w.h_lp.size() * 8, cudaMemcpyDeviceToHost);
      w.finished = true;
    }
    return active;
  }
  // tokens of live slot m after step t (back-pointers, decoding.py:114 child.tokens)
  int beam_path(int b, int t, int m, int* tokens, int cap) {
    const BeamWs& w = bw;
    const int n = t + 1;
    if (n > cap) throw Error(CMT_ERR_SHAPE, "token buffer too small");
    for (int q = t; q >= 0; --q) {
      const int2 e = w.h_bp[((size_t)b * w.Tmax + q) * w.K + m];
      tokens[q] = e.y;
      m = e.x;
    }
    return n;
  }
  // result `rank` of sentence b: finished hypotheses best first (score desc,
  // arrival asc), tokens without the EOS; or the truncation fallback
  int beam_result(int b, int rank, int* tokens, int cap, int* n_tok, double* score, double* logp, int* trunc) {
    const BeamWs& w = bw;
    if (!w.finished) throw Error(CMT_ERR_CONFIG, "beam search still running");
    if (b < 0 || b >= w.B) throw Error(CMT_ERR_SHAPE, "sentence index out of range");
    const BeamSent& q = w.h_sent[b];
    const int count = q.nf > 0 ? std::min(q.nf, w.nb) : 1;
    if (rank < 0 || rank >= count) throw Error(CMT_ERR_SHAPE, "result rank out of range");
    if (q.nf > 0) {
      const BeamFin& f = w.h_fin[(size_t)b * w.nb + rank];
      *n_tok = f.t > 0 ? beam_path(b, f.t - 1, f.parent, tokens, cap) : 0;
      *score = f.score;
      *logp = f.logp;
      *trunc = 0;
    } else {
      *n_tok = q.t > 0 ? beam_path(b, q.t - 1, q.trunc_slot, tokens, cap) : 0;
      *logp = w.h_lp[(size_t)b * w.K + q.trunc_slot];
      *score = NAN;  // log_prob / lp(max(len, 1)): computed by the caller (decoding.py:150-153)
      *trunc = 1;
    }
    return count;
  }

  // ---- workspace carving for (S, T, B) ----
  template <typename P>
  P* carve(char*& cur, size_t bytes) {
    P* p = (P*)cur;
    cur += (bytes + 255) & ~(size_t)255;
    return p;
  }
  size_t layout(char* base) {
    char* cur = base;
    long long NS = (long long)S * B, NT = (long long)T * B;
    long long Nmax = std::max(NS, NT);
    int nl = (int)layers.size();
    lw.assign(nl, {});
    for (int l = 0; l < nl; ++l) {
      long long steps = (l <= L) ? S : T;  // layers 0..L are encoder
      long long N = steps * B;
      lw[l].yext = carve<char>(cur, (steps + 1) * B * H * asz);
      lw[l].cext = carve<float>(cur, (steps + 1) * B * H * 4);
      lw[l].acts = carve<float>(cur, N * 4 * H * 4);
      lw[l].tc = carve<float>(cur, N * H * 4);
      lw[l].dy = carve<float>(cur, N * H * 4);
    }
    src_ids_d = carve<int>(cur, NS * 4);
    tgt_in_d = carve<int>(cur, NT * 4);
    tgt_out_d = carve<int>(cur, NT * 4);
    src_mask_d = carve<float>(cur, NS * 4);
    tgt_mask_d = carve<float>(cur, NT * 4);
    Xs = carve<char>(cur, NS * E * asz);
    Xt = carve<char>(cur, NT * E * asz);
    top = carve<char>(cur, NS * H * asz);
    ux = carve<float>(cur, Nmax * 4 * H * 4);
    ux2 = carve<float>(cur, Nmax * 4 * H * 4);
    ux3 = carve<float>(cur, NT * 4 * H * 4);  // dec.l1 input projection, computed early (see run())
    dU = carve<char>(cur, Nmax * 4 * H * asz);
    dU2 = carve<char>(cur, Nmax * 4 * H * asz);
    dUl.assign(layers.size(), nullptr);
    if (bwd_split_mem())
      for (size_t l = 0; l < layers.size(); ++l) dUl[l] = carve<char>(cur, (long long)(l <= (size_t)L ? NS : NT) * 4 * H * asz);
    drop_enc.assign(L + 1, nullptr); keep_enc.assign(L + 1, nullptr);
    drop_dec.assign(L + 1, nullptr); keep_dec.assign(L + 1, nullptr);
    for (int k = 2; k <= L; ++k) {
      drop_enc[k] = carve<char>(cur, NS * H * asz);
      keep_enc[k] = carve<uint8_t>(cur, NS * H);
      drop_dec[k] = carve<char>(cur, NT * H * asz);
      keep_dec[k] = carve<uint8_t>(cur, NT * H);
    }
    u_att = carve<char>(cur, NT * H * asz);
    alpha = carve<float>(cur, (long long)B * T * S * 4);
    att_dsc = carve<float>(cur, (long long)B * T * S * 4);
    att_part = att_tc_ok() ? nullptr
                           : carve<float>(cur, (long long)B * att::nslices(H) * att2::tiles(T) * att2::tiles(S) * att2::P *
                                                   att2::P * 4);
    if (att_tc_ok()) {  // bf16 alpha / dscores [B][T][S8] and dC [N_T][H] for the tcgen05 attention
      att_a16 = carve<bf16>(cur, (long long)B * T * s8() * 2);
      att_d16 = carve<bf16>(cur, (long long)B * T * s8() * 2);
      att_dc16 = carve<bf16>(cur, NT * H * 2);
    }
    cst_att = carve<char>(cur, NT * 2 * H * asz);
    ho = carve<float>(cur, NT * H * 4);
    hod = carve<char>(cur, NT * H * asz);
    keep_o = carve<uint8_t>(cur, NT * H);
    Y = carve<char>(cur, NT * (long long)V * asz);
    losstok = carve<float>(cur, NT * 4);
    dhpre = carve<char>(cur, NT * H * asz);
    dho32 = bf ? carve<float>(cur, NT * H * 4) : nullptr;
    dcst = carve<float>(cur, NT * 2 * H * 4);
    du_att = carve<char>(cur, NT * H * asz);
    dXemb = carve<float>(cur, (NS + NT) * E * 4);
    dtop = carve<float>(cur, NS * H * 4);
    dhc = carve<float>(cur, (long long)B * H * 4);
    dcc = carve<float>(cur, (long long)B * H * 4);
    fin_dh.assign(L + 1, nullptr); fin_dc.assign(L + 1, nullptr);
    for (int k = 1; k <= L; ++k) {
      fin_dh[k] = carve<float>(cur, (long long)B * H * 4);
      fin_dc[k] = carve<float>(cur, (long long)B * H * 4);
    }
    long long colmax = std::max<long long>(V, 4LL * H);
    colpart = carve<float>(cur, 64 * colmax * 4);
    colpart2 = carve<float>(cur, 64 * colmax * 4);
    colticket = carve<unsigned>(cur, 2 * 1024 * 4);
    colticket2 = colticket + 1024;
    if (base) CMT_CUDA(cudaMemsetAsync(colticket, 0, 2 * 1024 * 4, st));
    cepart = use_ce2() ? carve<float>(cur, std::max<long long>(g_num_sms, ceil_div(NT, CEG_ROWS)) * V * 4) : nullptr;
    cerow = carve<float2>(cur, (size_t)NT * 8);
    for (int t = 0; t < 2; ++t) {
      seg_off_d[t] = carve<int>(cur, (NS + NT + 1) * 4);
      seg_pos_d[t] = carve<int>(cur, (NS + NT) * 4);
      uniq_d[t] = carve<int>(cur, (NS + NT) * 4);
      gcomp[t] = carve<float>(cur, (NS + NT) * E * 4);
    }
    normpart = carve<double>(cur, (2 * layers.size() + 8) * NORM_BLOCKS * 8);
    flags = carve<unsigned>(cur, flag_words() * 4);
    scal_d = carve<StepScalars>(cur, sizeof(StepScalars));
    out_d = carve<StepOut>(cur, sizeof(StepOut));
    s32_d = carve<float>(cur, 4);
    return (size_t)(cur - base);
  }
  void ensure_ws(int S_, int T_, int B_) {
    S = S_; T = T_; B = B_;
    size_t need = layout(nullptr);
    if (need > ws_cap) {
      CMT_CUDA(cudaStreamSynchronize(st));
      drop_graphs();  // captured steps point into the old workspace
      if (ws) cudaFree(ws);
      ws = nullptr;
      CMT_CUDA(cudaMalloc(&ws, need));
      ws_cap = need;
    }
    layout(ws);
    status_d = &out_d->status;
    losssum_d = &out_d->loss_sum;
    normscal_d = out_d->scal;
  }

  // ---- batch staging: host validation (model.py:146-151, attention.py:153-154) + H2D ----
  void stage(const long long* src, const float* smask, int S_, const long long* tgt, const float* tmask, int T_,
             int B_) {
    if (S_ < 1 || T_ < 1 || B_ < 1) throw Error(CMT_ERR_SHAPE, "batch dimensions must be positive");
    auto tick = [&](int i) {
      static thread_local std::chrono::steady_clock::time_point t0;
      auto t1 = std::chrono::steady_clock::now();
      if (i > 0) stage_us[i - 1] += std::chrono::duration<double, std::micro>(t1 - t0).count();
      t0 = t1;
    };
    tick(0);
    auto bad_id = [&](const long long* ids, long long n, long long& bad) {
      for (long long i = 0; i < n; ++i)
        if (ids[i] < 0 || ids[i] >= V) { bad = ids[i]; return true; }
      return false;
    };
    long long bad;
    long long NS = (long long)S_ * B_, NT = (long long)T_ * B_;
    if (bad_id(src, NS, bad) || bad_id(tgt, NT, bad))
      throw Error(CMT_ERR_CONFIG, "token id " + std::to_string(bad) + " outside vocabulary of size " + std::to_string(V));
    for (int b = 0; b < B_; ++b) {
      bool any = false;
      for (int s = 0; s < S_; ++s) any |= smask[(long long)s * B_ + b] > 0.f;
      if (!any) throw Error(CMT_ERR_MASK, "a batch column has every source position masked");
    }
    float ntok = 0.f;  // numpy float32 sum of {0,1} masks is exact below 2^24
    for (long long i = 0; i < NT; ++i) ntok += tmask[i];
    ntok_local = ntok;
    if (!(ntok > 0.f) && !allow_empty_targets)
      throw Error(CMT_ERR_CONFIG, "smoothed_loss needs at least one unmasked token");
    tick(1);
    ensure_ws(S_, T_, B_);
    tick(2);
    // pinned staging: ids (int32) + masks + segments
    size_t nbytes = (size_t)(NS + 2 * NT) * 4 + (size_t)(NS + NT) * 4 + 2 * (size_t)(3 * (NS + NT) + 2) * 4;
    // two pinned buffers: this batch's host work (conversion, segment sort)
    // overlaps the step still running on the device; only the copies issued
    // from the same buffer two batches ago must have landed
    const int k = pin_cur ^= 1;
    CMT_CUDA(cudaEventSynchronize(pin_ev[k]));
    char* p = (char*)pin_in[k].get(nbytes);
    int* h_src = (int*)p;
    int* h_tin = h_src + NS;
    int* h_tout = h_tin + NT;
    float* h_sm = (float*)(h_tout + NT);
    float* h_tm = h_sm + NS;
    for (long long i = 0; i < NS; ++i) h_src[i] = (int)src[i];
    for (int b = 0; b < B_; ++b) h_tin[b] = 2;  // BOS (model.py:239-244)
    for (long long i = B_; i < NT; ++i) h_tin[i] = (int)tgt[i - B_];
    for (long long i = 0; i < NT; ++i) h_tout[i] = (int)tgt[i];
    std::memcpy(h_sm, smask, NS * 4);
    std::memcpy(h_tm, tmask, NT * 4);
    CMT_CUDA(cudaMemcpyAsync(src_ids_d, h_src, NS * 4, cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(tgt_in_d, h_tin, NT * 4, cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(tgt_out_d, h_tout, NT * 4, cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(src_mask_d, h_sm, NS * 4, cudaMemcpyHostToDevice, st));
    CMT_CUDA(cudaMemcpyAsync(tgt_mask_d, h_tm, NT * 4, cudaMemcpyHostToDevice, st));
    tick(3);
    // embedding segments: unique ids (ascending) with their positions in order
    int* q = (int*)(h_tm + NT);
    // (id, position) pairs grouped by id, positions ascending within an id
    // (= np.add.at order): the keys are built in position order and an LSD
    // radix sort is stable, so sorting on the id bits alone (11-bit digits:
    // two passes for V <= 2^22) keeps the positions ascending within an id
    auto build = [&](int t, std::vector<unsigned long long>& keys) {
      const int n = (int)keys.size();
      sort_tmp.resize(n);
      unsigned long long* src_k = keys.data();
      unsigned long long* dst_k = sort_tmp.data();
      for (int shift = 32; shift < 64 && ((unsigned long long)(V - 1) >> (shift - 32)); shift += 11) {
        unsigned cnt[2049];
        std::memset(cnt, 0, sizeof(cnt));
        for (int i = 0; i < n; ++i) ++cnt[((src_k[i] >> shift) & 2047) + 1];
        for (int d = 0; d < 2048; ++d) cnt[d + 1] += cnt[d];
        for (int i = 0; i < n; ++i) dst_k[cnt[(src_k[i] >> shift) & 2047]++] = src_k[i];
        std::swap(src_k, dst_k);
      }
      int* off = q; int* pos = q + n + 1; int* uq = pos + n;
      int nu = 0;
      for (int i = 0; i < n; ++i) {
        const int id = (int)(src_k[i] >> 32);
        if (i == 0 || id != (int)(src_k[i - 1] >> 32)) { off[nu] = i; uq[nu] = id; ++nu; }
        pos[i] = (int)(src_k[i] & 0xffffffffull);
      }
      off[nu] = n;
      nuniq[t] = nu;
      nrows_max[t] = std::min(n, V);
      nseg_pos[t] = n;
      uniq_h[t].assign(uq, uq + nu);
      CMT_CUDA(cudaMemcpyAsync(seg_off_d[t], off, (nu + 1) * 4, cudaMemcpyHostToDevice, st));
      CMT_CUDA(cudaMemcpyAsync(seg_pos_d[t], pos, n * 4, cudaMemcpyHostToDevice, st));
      CMT_CUDA(cudaMemcpyAsync(uniq_d[t], uq, nu * 4, cudaMemcpyHostToDevice, st));
      q = uq + nu;
    };
    const long long nmax_t = cfg.shared_embeddings ? NS + NT : std::max(NS, NT);
    seg_dev = use_seg_dev && !comm && nmax_t <= SEG_MAX_N;
    tick(4);
    if (seg_dev) {  // built by segments_kernel inside the step; host copies of the ids for host-side readers
      seg_ids_h[0].assign(h_src, h_src + NS);
      if (cfg.shared_embeddings) seg_ids_h[0].insert(seg_ids_h[0].end(), h_tin, h_tin + NT);
      else seg_ids_h[1].assign(h_tin, h_tin + NT);
      for (int t = 0; t < 2; ++t) {
        const long long n = t == 0 ? (cfg.shared_embeddings ? NS + NT : NS) : (cfg.shared_embeddings ? 0 : NT);
        nrows_max[t] = (int)std::min<long long>(n, V);
        nseg_pos[t] = (int)n;
        nuniq[t] = nrows_max[t];  // upper bound; the step reads the count from the device
        seg_host_ok[t] = false;
        uniq_h[t].clear();
      }
      tick(5);
      CMT_CUDA(cudaEventRecord(pin_ev[k], st));
      tick(6);
      stage_us[7] += 1;
      staged = true;
      union_set[0] = union_set[1] = false;
      return;
    }
    std::vector<unsigned long long> ka, kb;
    ka.reserve(NS + NT);
    kb.reserve(NT);
    for (long long i = 0; i < NS; ++i) ka.push_back(((unsigned long long)h_src[i] << 32) | (unsigned)i);
    for (long long i = 0; i < NT; ++i) kb.push_back(((unsigned long long)h_tin[i] << 32) | (unsigned)(NS + i));
    seg_host_ok[0] = seg_host_ok[1] = true;
    if (cfg.shared_embeddings) {
      ka.insert(ka.end(), kb.begin(), kb.end());
      build(0, ka);
      nuniq[1] = 0;
      nrows_max[1] = 0;
    } else {
      build(0, ka);
      build(1, kb);
    }
    tick(5);
    CMT_CUDA(cudaEventRecord(pin_ev[k], st));
    tick(6);
    stage_us[7] += 1;
    staged = true;
    union_set[0] = union_set[1] = false;  // a new batch: its rows union comes with it
  }

  // ---- launch helpers ----
  template <class Epi>
  void gemm(int M, int N, int K, Mat A, Mat Bm, const Epi& e, int bn = 0) {
    if (M <= 0 || N <= 0) return;
    if (!bf) {
      dim3 grid(ceil_div(N, 64), ceil_div(M, 64));
      gemm_simt_kernel<Epi><<<grid, 256, 0, st>>>((const float*)A.p, A.ld, A.mn, (const float*)Bm.p, Bm.ld, Bm.mn, M,
                                                   N, K, e);
      CMT_LAUNCHED(); tl_mark(st, "gemm_simt_kernel");
      CMT_CUDA(cudaGetLastError());
      return;
    }
    if (K < tc::BK) {
      // tiny contraction (toy dims / K=0 BPTT start): TMA boxes would exceed the
      // tensor extent, run the bf16 SIMT kernel with the same epilogue instead
      dim3 grid(ceil_div(N, 64), ceil_div(M, 64));
      gemm_simt_kernel<Epi, bf16><<<grid, 256, 0, st>>>((const bf16*)A.p, A.ld, A.mn, (const bf16*)Bm.p, Bm.ld, Bm.mn,
                                                          M, N, K, e);
      CMT_LAUNCHED(); tl_mark(st, "gemm_simt_kernel");
      CMT_CUDA(cudaGetLastError());
      return;
    }
    dispatch_tc(M, N, K, A, Bm, e, bn);
  }
  void dispatch_tc(int M, int N, int K, Mat A, Mat Bm, const EpiStore& e, int bn) {
    int tile = bn ? bn * 4 + 1 : pick_tile(M, N);
    if (!cg2 && (tile & 3) == 2) tile = (tile >> 2) * 4 + 1;
    int key = A.mn * 2 + Bm.mn;
#define CMT_TC(BN_, AMN, BMN, CG_) \
  if (tile == BN_ * 4 + CG_ && key == AMN * 2 + BMN) return launch_tc<BN_, AMN, BMN, EpiStore, CG_>(st, M, N, K, A, Bm, e);
    CMT_TC(64, 0, 1, 1) CMT_TC(128, 0, 1, 1) CMT_TC(256, 0, 1, 1)
    CMT_TC(64, 0, 0, 1) CMT_TC(128, 0, 0, 1) CMT_TC(256, 0, 0, 1)
    CMT_TC(64, 1, 1, 1) CMT_TC(128, 1, 1, 1) CMT_TC(256, 1, 1, 1)
    CMT_TC(128, 0, 1, 2) CMT_TC(256, 0, 1, 2)
    CMT_TC(128, 0, 0, 2) CMT_TC(256, 0, 0, 2)
    CMT_TC(128, 1, 1, 2) CMT_TC(256, 1, 1, 2)
#undef CMT_TC
    throw Error(CMT_ERR_INTERNAL, "no tcgen05 GEMM instantiation for this operand layout");
  }
  void dispatch_tc(int M, int N, int K, Mat A, Mat Bm, const EpiLstmFwd& e, int) {
    if (A.mn || !Bm.mn) throw Error(CMT_ERR_INTERNAL, "lstm fwd layout");
    launch_tc<64, 0, 1, EpiLstmFwd>(st, M, N, K, A, Bm, e);
  }
  void dispatch_tc(int M, int N, int K, Mat A, Mat Bm, const EpiLstmBwd& e, int) {
    if (A.mn || Bm.mn) throw Error(CMT_ERR_INTERNAL, "lstm bwd layout");
    launch_tc<32, 0, 0, EpiLstmBwd>(st, M, N, K, A, Bm, e);
  }
  void dispatch_tc(int M, int N, int K, Mat A, Mat Bm, const EpiInitGrad& e, int) {
    launch_tc<32, 0, 0, EpiInitGrad>(st, M, N, K, A, Bm, e);
  }

  EpiStore store(void* C, long long ldc, bool c_act) const {
    EpiStore e;
    e.C = C; e.ldc = ldc; e.c_bf16 = (c_act && bf) ? 1 : 0;
    return e;
  }
  int grid_for(long long n) const { return (int)std::min<long long>(8 * g_num_sms, std::max<long long>(1, ceil_div(n, 256))); }

  template <typename T>
  void launch_gather(const void* table, const int* ids, int N, void* out) {
    gather_rows_kernel<T><<<N, 128, 0, st>>>((const T*)table, E, ids, N, (T*)out);
    CMT_LAUNCHED(); tl_mark(st, "gather_rows_kernel");
  }
  void gather(int t, const int* ids, int N, void* out) {
    if (bf) launch_gather<bf16>(table_v(t), ids, N, out);
    else launch_gather<float>(table_v(t), ids, N, out);
  }
  PcgJump* jump_d = nullptr;  // PCG64 jump-ahead table for jump_inc
  unsigned long long jump_inc[2] = {0, 0};
  bool jump_ok = false;
  void ensure_jump(const Pcg& pcg) {
    if (jump_ok && jump_inc[0] == pcg.inc_hi && jump_inc[1] == pcg.inc_lo) return;
    if (!jump_d) CMT_CUDA(cudaMalloc(&jump_d, sizeof(PcgJump)));
    pcg_jump_table_kernel<<<1, 1, 0, st>>>(jump_d, pcg.inc_hi, pcg.inc_lo);
    CMT_LAUNCHED(); tl_mark(st, "pcg_jump_table_kernel");
    jump_inc[0] = pcg.inc_hi; jump_inc[1] = pcg.inc_lo;
    jump_ok = true;
  }
  // dropout site (layers.py:265-296): numpy-exact PCG64 draws by jump-ahead;
  // x2 (optional) is added to x first (the bidirectional sum feeding enc.l2)
  template <typename TI, typename TO>
  void launch_dropout(const void* x, void* y, uint8_t* keep, int N, unsigned long long base, const Pcg* pcg,
                      const void* x2 = nullptr) {
    if (!jump_ok) throw Error(CMT_ERR_INTERNAL, "PCG64 jump table not built");
    dim3 blk(32, 8);
    dim3 grid(ceil_div(H, 32), ceil_div(ceil_div(N, DROP4_DPT), 8));
    float scale = 1.0f / (float)(1.0 - cfg.dropout);
    ncu_begin(8);
    dropout_fwd_kernel4<TI, TO><<<grid, blk, 0, st>>>((const TI*)x, (TO*)y, keep, N, H, pcg, jump_d, base,
                                                      dropout_threshold(cfg.dropout), scale, (const TI*)x2);
    ncu_end();
    CMT_LAUNCHED(); tl_mark(st, "dropout_fwd_kernel4");
  }

  // masks queued for generation beside the next recurrent launch of scan_ctas
  // CTAs (one mask CTA per idle SM, on the side stream); ev_mask[id] marks each
  void flush_masks(int scan_ctas) {
    if (mask_queue.empty()) return;
    // side stream beside the scan; single-stream schedules (timeline) run them
    // on the main stream with the whole GPU
    const bool side = use_overlap();
    const int idle = side ? g_num_sms - scan_ctas : g_num_sms;
    if (idle < 1) throw Error(CMT_ERR_INTERNAL, "no idle SMs for the dropout masks");
    static bool attr = false;
    if (!attr) {
      CMT_CUDA(cudaFuncSetAttribute(dropout_mask_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DMASK_SMEM));
      attr = true;
    }
    auto gen = [&]() {
      for (const MaskSite& m : mask_queue) {
        ncu_begin(8);
        dropout_mask_kernel<<<idle, DMASK_THREADS, DMASK_SMEM, st>>>(m.keep, m.N, H, &scal_d->pcg, jump_d, m.base,
                                                                     dropout_threshold(cfg.dropout));
        ncu_end();
        CMT_LAUNCHED(); tl_mark(st, "dropout_mask_kernel");
        CMT_CUDA(cudaEventRecord(ev_mask[m.id], st));
      }
    };
    if (side) {
      fork();
      on_side_stream(gen);
    } else {
      gen();
    }
    mask_queue.clear();
  }
  // a site whose mask was generated ahead: wait for it, then y = x * keep / (1 - p)
  template <typename TI, typename TO>
  void apply_dropout(int id, const void* x, const void* x2, const uint8_t* keep, void* y, long long n) {
    CMT_CUDA(cudaStreamWaitEvent(st, ev_mask[id], 0));
    const float scale = 1.0f / (float)(1.0 - cfg.dropout);
    ncu_begin(13);
    dropout_apply_kernel<TI, TO><<<grid_for(n / 8), 256, 0, st>>>((const TI*)x, (const TI*)x2, keep, (TO*)y, n,
                                                                  scale);
    ncu_end();
    CMT_LAUNCHED(); tl_mark(st, "dropout_apply_kernel");
  }

  // ---- persistent recurrent kernels (bf16) ----
  // ---- LSTM scans ----
  struct ScanViews {
    void* ybase;        // y[0]
    const void* hprev;  // h_{t-1} for t (row t*B+b)
    float* cbase;
    const float* cprev;
  };
  ScanViews views(int l, bool reverse) {
    long long slot = (long long)B * H;
    char* y = (char*)lw[l].yext;
    float* c = lw[l].cext;
    if (!reverse) return {y + slot * asz, y, c + slot, c};
    return {y, y + slot * asz, c, c + slot};
  }

  // ---- paired forward scans (lstm_multi.cuh) ----
  struct FwdScan {
    int l;
    const void* X;
    int din, steps;
    bool reverse;
    const float* mask;
    float* uxb;  // hoisted input projection buffer of this scan
  };
  template <int ROWS>
  bool fwd_multi_ok() const {
    using F = mc::Fwd<ROWS>;
    const int nh = (B + ROWS - 1) / ROWS;
    return bf && persistent && dual && H % (64 * F::KBOX) == 0 && H / 64 <= 32 && (H / 64) * nh <= FLAG_STRIDE &&
           F::ctas(H, B) <= g_num_sms && F::stages(H) >= 2;
  }
  template <int ROWS>
  bool fwd_tm_ok() const {
    using F = tm::Fwd<ROWS>;
    const int nh = (B + ROWS - 1) / ROWS;
    return bf && persistent && fwd_tm && F::ok(H, B) && H / 64 <= 32 && (H / 64) * nh <= FLAG_STRIDE &&
           F::ctas(H, B) <= g_num_sms;
  }
  bool dual_tm() const { return dual && fwd_tm_ok<64>() && 2 * tm::Fwd<64>::ctas(H, B) <= g_num_sms; }
  bool use_dual_fwd() const {
    return dual_tm() || (fwd_multi_ok<128>() && 2 * mc::Fwd<128>::ctas(H, B) <= g_num_sms);
  }
  void fwd_prep(const FwdScan& f) {  // Ux = X W_x + b (layers.py:354-357, K3)
    const Layer& ly = layers[f.l];
    EpiStore e = store(f.uxb, 4LL * H, false);
    e.bias = dw + ly.b_off;
    ncu_begin(3);
    gemm(f.steps * B, 4 * H, f.din, Mat{f.X, f.din, 0}, Mat{wv(ly.w_off), 4LL * H, 1}, e);
    ncu_end();
  }
  template <int ROWS>
  LstmFwdP fwd_params(const FwdScan& f, CUtensorMap* tmH, CUtensorMap* tmW) {
    const Layer& ly = layers[f.l];
    ScanViews v = views(f.l, f.reverse);
    make_map_kblocks(tmH, lw[f.l].yext, (long long)(f.steps + 1) * B, H, H, ROWS, mc::Fwd<ROWS>::KBOX);
    make_map(tmW, wv(ly.w_off), 4LL * H, f.din + H, 4LL * H, 64, 64);
    LstmFwdP prm;
    prm.ux = f.uxb; prm.y = (bf16*)v.ybase; prm.hprev = (const bf16*)v.hprev; prm.cst = v.cbase; prm.cprev = v.cprev;
    prm.acts = lw[f.l].acts; prm.tcache = lw[f.l].tc; prm.mask = f.mask; prm.flag = fwd_flags(f.l); prm.status = status_d;
    prm.steps = f.steps; prm.B = B; prm.H = H; prm.din = f.din; prm.reverse = f.reverse ? 1 : 0;
    prm.hrow0 = f.reverse ? B : 0;
    prm.trace = (trace_layer == f.l) ? trace_d : nullptr;
    prm.stages = mc::Fwd<ROWS>::stages(H);
    return prm;
  }
  // lstm_fwd_tm<ROWS>: one or two scans per cooperative launch
  template <int ROWS>
  void fwd_tm_launch(const FwdScan& a, const FwdScan* b) {
    using F = tm::Fwd<ROWS>;
    CUtensorMap tmap[4];
    LstmFwdMulti m;
    auto prm = [&](const FwdScan& f, CUtensorMap* tmH, CUtensorMap* tmW) {
      LstmFwdP r = fwd_params<128>(f, tmH, tmW);
      make_map_kblocks(tmH, lw[f.l].yext, (long long)(f.steps + 1) * B, H, H, ROWS, F::KBOX);
      r.stages = F::stages(H);
      return r;
    };
    m.c[0] = prm(a, &tmap[0], &tmap[1]);
    if (b) m.c[1] = prm(*b, &tmap[2], &tmap[3]);
    else { m.c[1] = m.c[0]; tmap[2] = tmap[0]; tmap[3] = tmap[1]; }
    const int g = F::ctas(H, B);
    m.split = g;
    auto k = lstm_fwd_tm<ROWS>;
    const size_t smem = F::smem(H);
    CMT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(b ? 2 * g : g);
    c.blockDim = dim3(tm::THREADS);
    c.dynamicSmemBytes = smem;
    c.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = g_coop;
    c.attrs = at;
    c.numAttrs = 1;
    flush_masks(c.gridDim.x);
    cudaEvent_t p0 = probe_begin(2);
    CMT_CUDA(cudaLaunchKernelEx(&c, k, tmap[0], tmap[1], tmap[2], tmap[3], m));
    probe_end(2, p0);
    CMT_LAUNCHED();
    tl_mark(st, b ? "lstm_fwd_tm_pair" : "lstm_fwd_tm_single");
  }
  // two independent scans in one cooperative launch (64 CTAs each at H=1024, B=128)
  void fwd_pair(const FwdScan& a, const FwdScan& b) {
    if (dual_tm()) return fwd_tm_launch<64>(a, &b);
    CUtensorMap tm[4];
    LstmFwdMulti m;
    m.c[0] = fwd_params<128>(a, &tm[0], &tm[1]);
    m.c[1] = fwd_params<128>(b, &tm[2], &tm[3]);
    const int g = mc::Fwd<128>::ctas(H, B);
    m.split = g;
    auto k = lstm_fwd_multi<128>;
    const size_t smem = mc::Fwd<128>::smem(H);
    CMT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(2 * g);
    c.blockDim = dim3(mc::THREADS);
    c.dynamicSmemBytes = smem;
    c.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = g_coop;
    c.attrs = at;
    c.numAttrs = 1;
    flush_masks(c.gridDim.x);
    cudaEvent_t p0 = probe_begin(2);
    CMT_CUDA(cudaLaunchKernelEx(&c, k, tm[0], tm[1], tm[2], tm[3], m));
    probe_end(2, p0);
    CMT_LAUNCHED();
    tl_mark(st, "lstm_fwd_pair");
  }

  // one scan through lstm_fwd_multi<ROWS>: batch slices of ROWS rows on separate
  // CTAs (ROWS=64: 128 CTAs at H=1024, B<=128; ROWS=128: B<=256)
  int single_fwd_rows() const { return fwd_multi_ok<64>() ? 64 : fwd_multi_ok<128>() ? 128 : 0; }
  template <int ROWS>
  void fwd_single(const FwdScan& a) {
    CUtensorMap tm[2];
    LstmFwdMulti m;
    m.c[0] = fwd_params<ROWS>(a, &tm[0], &tm[1]);
    m.c[1] = m.c[0];
    const int g = mc::Fwd<ROWS>::ctas(H, B);
    m.split = g;
    auto k = lstm_fwd_multi<ROWS>;
    const size_t smem = mc::Fwd<ROWS>::smem(H);
    CMT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(g);
    c.blockDim = dim3(mc::THREADS);
    c.dynamicSmemBytes = smem;
    c.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = g_coop;
    c.attrs = at;
    c.numAttrs = 1;
    flush_masks(c.gridDim.x);
    cudaEvent_t p0 = probe_begin(2);
    CMT_CUDA(cudaLaunchKernelEx(&c, k, tm[0], tm[1], tm[0], tm[1], m));
    probe_end(2, p0);
    CMT_LAUNCHED();
    tl_mark(st, "lstm_fwd_single");
  }

  void scan_fwd(int l, const void* X, int din, int steps, bool reverse, const float* mask) {
    // single scans: lstm_fwd_multi<64> (128 CTAs, 6.4 us/step at c3) beats the
    // TMEM-split kernel with 32-row slices (6.9 us/step), but when the batch
    // needs 128-row multi slices (B > 128) the TMEM-split kernel with 64-row
    // slices is faster (c5: 28.5 -> 28.2 ms/step)
    if (fwd_tm == 1 && single_fwd_rows() == 128 && fwd_tm_ok<64>()) {
      FwdScan f{l, X, din, steps, reverse, mask, ux};
      fwd_prep(f);
      fwd_tm_launch<64>(f, nullptr);
      return;
    }
    if (const int rows = single_fwd_rows()) {
      FwdScan f{l, X, din, steps, reverse, mask, ux};
      fwd_prep(f);
      if (rows == 64) fwd_single<64>(f);
      else fwd_single<128>(f);
      return;
    }
    // general fallback (fp32 validation mode, shapes the persistent kernels do
    // not cover): the hoisted projection, then one GEMM per step with the cell
    // fused in its epilogue
    const Layer& ly = layers[l];
    // hoisted input projection Ux = X W_x + b   (layers.py:354-357, K3)
    EpiStore e = store(ux, 4LL * H, false);
    e.bias = dw + ly.b_off;
    gemm(steps * B, 4 * H, din, Mat{X, din, 0}, Mat{wv(ly.w_off), 4LL * H, 1}, e);
    ScanViews v = views(l, reverse);
    const void* Wh = (const char*)wv(ly.w_off) + (size_t)din * 4 * H * asz;
    for (int p = 0; p < steps; ++p) {
      int t = reverse ? steps - 1 - p : p;
      EpiLstmFwd f;
      f.ux = ux; f.hprev = v.hprev; f.cprev = v.cprev; f.y = v.ybase; f.cst = v.cbase;
      f.acts = lw[l].acts; f.tcache = lw[l].tc; f.mask = mask ? mask + (long long)t * B : nullptr;
      f.row0 = (long long)t * B; f.H = H; f.act_bf16 = bf;
      const void* hp = (const char*)v.hprev + (size_t)t * B * H * asz;
      gemm(B, 4 * H, H, Mat{hp, H, 0}, Mat{Wh, 4LL * H, 1}, f);
    }
  }

  // BPTT for layer l; writes dX (= or +=, optional dropout mask) and param grads.
  // ---- paired backward scans (lstm_multi.cuh) ----
  struct BwdScan {
    int l;
    const void* X;
    int din, steps;
    bool reverse;
    const float* mask;
    const float* dy;
    const float* dh_final;
    const float* dc_final;
    float* dh0;
    float* dc0;
    float* dX;
    int dx_beta;
    const uint8_t* dx_keep;
    void* dUb;
  };
  // BPTT cluster K-split: 4 CTAs per 64 units.  (A split of 8 halves each
  // CTA's dU stream and doubles its TMA stages in flight, but only 15 clusters
  // of 8 are co-resident on this B200 against the 16 a scan pair needs.)
  static constexpr int BWD_KS = 4;
  template <int ROWS>
  bool bwd_multi_ok() const {
    using F = mc::Bwd<ROWS, BWD_KS>;
    const int kbl = 4 * H / 64 / BWD_KS;
    return bf && persistent && dual && H % mc::BWD_NU == 0 && (4 * H / 64) % BWD_KS == 0 &&
           kbl % mc::BWD_KBOX == 0 && kbl <= 32 && (4 * H / 64) * ((B + ROWS - 1) / ROWS) <= FLAG_STRIDE &&
           F::ctas(H, B) <= g_num_sms && F::stages(H) >= 2 && (size_t)F::stages(H) * F::STAGE >= F::xbuf_bytes();
  }
  template <int ROWS>
  int bwd_ctas() const { return mc::Bwd<ROWS, BWD_KS>::ctas(H, B); }
  bool use_dual_bwd() const { return bwd_multi_ok<128>() && 2 * bwd_ctas<128>() <= g_num_sms; }
  // one scan over batch slices of ROWS rows (64: two halves of B<=128; 128: B<=256)
  int single_bwd_rows() const { return bwd_multi_ok<64>() ? 64 : bwd_multi_ok<128>() ? 128 : 0; }
  void bwd_single(const BwdScan& f, bool post = true) {
    if (single_bwd_rows() == 64) bwd_launch<64>(f, nullptr);
    else bwd_launch<128>(f, nullptr);
    if (post) bwd_post(f);
  }
  template <int ROWS, int KS>
  LstmBwdP bwd_params(const BwdScan& f, CUtensorMap* tmA, CUtensorMap* tmW) {
    const Layer& ly = layers[f.l];
    ScanViews v = views(f.l, f.reverse);
    long long N = (long long)f.steps * B;
    make_map_kblocks(tmA, f.dUb, N, 4LL * H, 4LL * H, ROWS, mc::BWD_KBOX);
    make_map(tmW, wv(ly.w_off), 4LL * H, f.din + H, 4LL * H, 64, mc::BWD_NU);
    LstmBwdP prm;
    prm.dy = f.dy; prm.acts = lw[f.l].acts; prm.tcache = lw[f.l].tc; prm.cprev = v.cprev; prm.mask = f.mask;
    prm.dU = (bf16*)f.dUb; prm.dh_final = f.dh_final; prm.dc_final = f.dc_final; prm.dh0 = f.dh0; prm.dc0 = f.dc0;
    prm.flag = bwd_flags(f.l);
    prm.status = status_d;
    prm.steps = f.steps; prm.B = B; prm.H = H; prm.din = f.din; prm.reverse = f.reverse ? 1 : 0;
    prm.trace = (trace_layer == 100 + f.l) ? trace_d : nullptr;
    prm.stages = mc::Bwd<ROWS, KS>::stages(H);
    return prm;
  }
  template <int ROWS, int KS = BWD_KS>
  void bwd_launch(const BwdScan& a, const BwdScan* b) {
    CUtensorMap tm[4];
    LstmBwdMulti m;
    m.c[0] = bwd_params<ROWS, KS>(a, &tm[0], &tm[1]);
    if (b) m.c[1] = bwd_params<ROWS, KS>(*b, &tm[2], &tm[3]);
    else { m.c[1] = m.c[0]; tm[2] = tm[0]; tm[3] = tm[1]; }
    const int g = mc::Bwd<ROWS, KS>::ctas(H, B);
    m.split = g;
    auto k = lstm_bwd_multi<ROWS, KS>;
    const size_t smem = mc::Bwd<ROWS, KS>::smem(H);
    CMT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(b ? 2 * g : g);
    c.blockDim = dim3(mc::Bwd<ROWS, KS>::THREADS);
    c.dynamicSmemBytes = smem;
    c.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = g_coop;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = KS;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    c.attrs = at;
    c.numAttrs = 2;
    cudaEvent_t p0 = probe_begin(1);
    CMT_CUDA(cudaLaunchKernelEx(&c, k, tm[0], tm[1], tm[2], tm[3], m));
    probe_end(1, p0);
    CMT_LAUNCHED();
    tl_mark(st, b ? "lstm_bwd_pair" : "lstm_bwd_single");
  }
  void bwd_pair(const BwdScan& a, const BwdScan& b) { bwd_launch<128>(a, &b); }
  // weight grads, bias grads and input grads of a finished BPTT scan
  void bwd_post(const BwdScan& f, int c0 = 0) {
    bwd_post_w(f, c0);
    if (f.dX) bwd_post_dx(f);
  }
  // weight and bias grads of a finished BPTT scan
  // dW[0:din] = X^T dU, dW[din:] = Hprev^T dU  (layers.py:389-391, batched; K6),
  // gate columns [c0, c1) of both halves
  void bwd_dw_cols(const BwdScan& f, int c0, int c1) {
    if (c1 <= c0) return;
    const Layer& ly = layers[f.l];
    ScanViews v = views(f.l, f.reverse);
    const long long N = (long long)f.steps * B;
    const void* du = (const char*)f.dUb + (size_t)c0 * asz;
    ncu_begin(5);
    gemm(f.din, c1 - c0, (int)N, Mat{f.X, f.din, 1}, Mat{du, 4LL * H, 1}, store(dg + ly.w_off + c0, 4LL * H, false));
    ncu_end();
    gemm(H, c1 - c0, (int)N, Mat{v.hprev, H, 1}, Mat{du, 4LL * H, 1},
         store(dg + ly.w_off + (size_t)f.din * 4 * H + c0, 4LL * H, false));
  }
  // the BPTT weight-gradient split: the first bg_cols() gate columns of a
  // level's dW run on the background stream beside the NEXT level's scans (on
  // the SMs those leave idle), the rest here at full width.  Off in data
  // parallel (the gradient buckets are all-reduced as levels finish) and in
  // the single-stream timeline.
  bool bwd_split_mem() const { return bf && bwd_bg > 0 && comm == nullptr && use_dual_bwd(); }
  bool bwd_split_ok() const { return bwd_split_mem() && !g_tl.on && !dUl.empty() && dUl[0] != nullptr; }
  int bg_cols() const { return bwd_split_ok() ? (4 * H * bwd_bg / 100) / 256 * 256 : 0; }
  int idle_sms() const { return g_num_sms - 2 * bwd_ctas<128>(); }
  void bwd_dw_bg(const BwdScan& f) {  // issue this level's deferred columns on the background stream
    const int nb = bg_cols();
    if (!nb || idle_sms() < 8) return;
    CMT_CUDA(cudaEventRecord(ev_bg, st));
    CMT_CUDA(cudaStreamWaitEvent(stb, ev_bg, 0));
    std::swap(st, stb);
    g_grid_cap = idle_sms() / 2 * 2;
    try {
      bwd_dw_cols(f, 0, nb);
    } catch (...) {
      std::swap(st, stb);
      g_grid_cap = 0;
      throw;
    }
    std::swap(st, stb);
    g_grid_cap = 0;
    bg_pending = true;
  }
  void bg_join() {
    if (!bg_pending) return;
    CMT_CUDA(cudaEventRecord(ev_bgj, stb));
    CMT_CUDA(cudaStreamWaitEvent(st, ev_bgj, 0));
    bg_pending = false;
  }
  void bwd_post_w(const BwdScan& f, int c0 = 0) {
    const Layer& ly = layers[f.l];
    long long N = (long long)f.steps * B;
    bwd_dw_cols(f, c0, 4 * H);
    colsum(f.dUb, true, N, 4 * H, dg + ly.b_off);
    allreduce_region(f.l);
  }
  // dX = dU W_x^T (layers.py:392; K7), dropout backward fused (layers.py:292-296)
  void bwd_post_dx(const BwdScan& f) {
    const Layer& ly = layers[f.l];
    long long N = (long long)f.steps * B;
    EpiStore e = store(f.dX, f.din, false);
    e.beta = f.dx_beta;
    if (f.dx_keep) { e.dmask = f.dx_keep; e.ld_dmask = f.din; e.dscale = 1.0f / (float)(1.0 - cfg.dropout); }
    ncu_begin(4);
    gemm((int)N, f.din, 4 * H, Mat{f.dUb, 4LL * H, 0}, Mat{wv(ly.w_off), 4LL * H, 0}, e);
    ncu_end();
  }

  void scan_bwd(int l, const void* X, int din, int steps, bool reverse, const float* mask, const float* dy,
                const float* dh_final, const float* dc_final, float* dh0, float* dc0, float* dX, int dx_beta,
                const uint8_t* dx_keep) {
    const Layer& ly = layers[l];
    long long N = (long long)steps * B;
    long long BH = (long long)B * H;
    ScanViews v = views(l, reverse);
    if (dh_final) CMT_CUDA(cudaMemcpyAsync(dhc, dh_final, BH * 4, cudaMemcpyDeviceToDevice, st));
    else CMT_CUDA(cudaMemsetAsync(dhc, 0, BH * 4, st));
    if (dc_final) CMT_CUDA(cudaMemcpyAsync(dcc, dc_final, BH * 4, cudaMemcpyDeviceToDevice, st));
    else CMT_CUDA(cudaMemsetAsync(dcc, 0, BH * 4, st));
    const void* WhN = (const char*)wv(ly.w_off) + (size_t)din * 4 * H * asz;  // rows din.. of [din+H][4H]
    auto time_of = [&](int p) { return reverse ? steps - 1 - p : p; };
    // general fallback: one GEMM per step with the cell backward in its epilogue
    for (int p = steps - 1; p >= 0; --p) {
      int t = time_of(p);
      EpiLstmBwd f;
      f.dy = dy; f.dhc = dhc; f.dc = dcc; f.acts = lw[l].acts; f.tcache = lw[l].tc; f.cprev = v.cprev;
      f.mask = mask ? mask + (long long)t * B : nullptr; f.dU = dU; f.row0 = (long long)t * B; f.H = H;
      f.act_bf16 = bf;
      if (p == steps - 1) {
        gemm(B, H, 0, Mat{nullptr, 4LL * H, 0}, Mat{WhN, 4LL * H, 0}, f);
      } else {
        int tn = time_of(p + 1);
        const void* a = (const char*)dU + (size_t)tn * B * 4 * H * asz;
        gemm(B, H, 4 * H, Mat{a, 4LL * H, 0}, Mat{WhN, 4LL * H, 0}, f);
      }
    }
    if (dh0) {
      EpiInitGrad f{dh0, dc0, dhc, dcc, H};
      const void* a = (const char*)dU + (size_t)time_of(0) * B * 4 * H * asz;
      gemm(B, H, 4 * H, Mat{a, 4LL * H, 0}, Mat{WhN, 4LL * H, 0}, f);
    }
    // weight grads: dW[0:din] = X^T dU, dW[din:] = Hprev^T dU  (layers.py:389-391, batched; K6)
    gemm(din, 4 * H, (int)N, Mat{X, din, 1}, Mat{dU, 4LL * H, 1}, store(dg + ly.w_off, 4LL * H, false));
    gemm(H, 4 * H, (int)N, Mat{v.hprev, H, 1}, Mat{dU, 4LL * H, 1},
         store(dg + ly.w_off + (size_t)din * 4 * H, 4LL * H, false));
    colsum(dU, true, N, 4 * H, dg + ly.b_off);
    // input grads dX = dU W_x^T (layers.py:392; K7), dropout backward fused (layers.py:292-296)
    EpiStore e = store(dX, din, false);
    e.beta = dx_beta;
    if (dx_keep) { e.dmask = dx_keep; e.ld_dmask = din; e.dscale = 1.0f / (float)(1.0 - cfg.dropout); }
    gemm((int)N, din, 4 * H, Mat{dU, 4LL * H, 0}, Mat{wv(ly.w_off), 4LL * H, 0}, e);
  }

  // ---- fork / join of the side stream ----
  bool use_overlap() const { return overlap && !g_tl.on; }  // the timeline measures one stream
  void fork() {
    CMT_CUDA(cudaEventRecord(ev_fork, st));
    CMT_CUDA(cudaStreamWaitEvent(st2, ev_fork, 0));
  }
  template <class F>
  void on_side_stream(F&& f) {  // issue f's launches on the side stream
    std::swap(st, st2);
    on_side = true;
    try {
      f();
    } catch (...) {
      std::swap(st, st2);
      on_side = false;
      throw;
    }
    std::swap(st, st2);
    on_side = false;
  }
  void join() {
    CMT_CUDA(cudaEventRecord(ev_join, st2));
    CMT_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
  }

  void colsum(const void* D, bool is_act, long long rows, int cols, float* out) {
    float* colpart = on_side ? colpart2 : this->colpart;
    unsigned* ticket = on_side ? colticket2 : colticket;
    int chunks = (int)std::min<long long>(64, std::max<long long>(1, rows / 64));
    int rows_per = ceil_div(rows, chunks);
    chunks = ceil_div(rows, rows_per);
    if (is_act && bf && cols % 8 == 0 && ceil_div(cols, 256) <= 1024) {  // 16-byte rows, fused final sum
      dim3 grid(ceil_div(cols, 256), chunks);
      colsum_partial_v8_kernel<<<grid, dim3(32, 8), 0, st>>>((const bf16*)D, cols, (int)rows, cols, rows_per, colpart,
                                                             ticket, out);
      CMT_LAUNCHED(); tl_mark(st, "colsum_v8_kernel");
      return;
    } else {
      dim3 grid(ceil_div(cols, 256), chunks);
      if (is_act && bf) colsum_partial_kernel<bf16><<<grid, 256, 0, st>>>((const bf16*)D, cols, (int)rows, cols, rows_per, colpart);
      else colsum_partial_kernel<float><<<grid, 256, 0, st>>>((const float*)D, cols, (int)rows, cols, rows_per, colpart);
    }
    CMT_LAUNCHED(); tl_mark(st, "colsum_partial_kernel");
    colsum_final_kernel<<<ceil_div(cols, 256), 256, 0, st>>>(colpart, chunks, cols, out);
    CMT_LAUNCHED(); tl_mark(st, "colsum_final_kernel");
  }

  template <typename T>
  void copy2d(const void* s, long long lds, void* d, long long ldd, int rows, int cols) {
    copy2d_kernel<T, T><<<grid_for((long long)rows * cols), 256, 0, st>>>((const T*)s, lds, (T*)d, ldd, rows, cols);
    CMT_LAUNCHED(); tl_mark(st, "copy2d_kernel");
  }
  void copy_act(const void* s, long long lds, void* d, long long ldd, int rows, int cols) {
    if (bf) copy2d<bf16>(s, lds, d, ldd, rows, cols);
    else copy2d<float>(s, lds, d, ldd, rows, cols);
  }

  // embedding grads of table t: deterministic segmented scatter of the dX rows
  // (tensor.py:208-216; np.add.at order) into compact rows, and in data
  // parallel the rows-union exchange (each table once per step)
  void embed_grads(int t, bool dp) {
    if (emb_sent[t]) return;
    emb_sent[t] = true;
    if (rows_grid(t)) {
      if (E % 4 == 0) {
        ncu_begin(12);
        scatter_compact_v4_kernel<<<rows_grid(t), SCAT_THREADS, 0, st>>>(dXemb, E, seg_off_d[t], seg_pos_d[t],
                                                                           nuniq[t], gcomp[t], rows_dev(t));
        ncu_end();
        CMT_LAUNCHED(); tl_mark(st, "scatter_compact_v4_kernel");
      } else {
        scatter_compact_kernel<<<rows_grid(t), 128, 0, st>>>(dXemb, E, seg_off_d[t], seg_pos_d[t], nuniq[t], gcomp[t],
                                                              rows_dev(t));
        CMT_LAUNCHED(); tl_mark(st, "scatter_compact_kernel");
      }
    }
    if (!dp) return;
    if (!union_set[t]) {
      if (world > 1) throw Error(CMT_ERR_CONFIG, "a data-parallel step needs the embedding rows union (cmt_set_union)");
      set_union(t, uniq_h[t].data(), nuniq[t]);  // one rank: the union is its own rows
    }
    if (!nunion[t]) return;
    CMT_CUDA(cudaMemsetAsync(ubuf[t], 0, (size_t)nunion[t] * E * 4, st));
    if (nuniq[t]) {
      scatter_rows_kernel<<<nuniq[t], 128, 0, st>>>(gcomp[t], E, umap_d[t], nuniq[t], ubuf[t]);
      CMT_LAUNCHED(); tl_mark(st, "scatter_rows_kernel");
    }
    allreduce(ubuf[t], (size_t)nunion[t] * E, NCCL_FLOAT32);
  }

  // ---- the step ----
  // One CUDA graph per (S, T, B, mode): the step's ~115 launches (recurrent
  // scans, GEMMs, CE, norm, update, side-stream forks) are captured the second
  // time a shape is run and replayed from then on.  Everything that varies
  // between batches of one shape is read from device memory: the step scalars
  // (generator state, lr, clip, smoothing, 1/ntok, embedding row counts;
  // set_scalars_kernel, launched before the graph) and the staged ids, masks
  // and segments.  Eager launches are kept for data parallelism (NCCL calls),
  // the timeline / probe / profiler-marker modes and debug early exits.
  struct ProbeNode {  // an event-record node of a captured probe (time_dominant)
    cudaGraphNode_t node;
    int pair;
    bool begin;
  };
  struct GraphEntry {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    unsigned long long draws = 0, kernels = 0;
    std::vector<ProbeNode> probe_nodes;
    std::vector<int> probe_cls;            // class of each captured probe pair
    std::vector<cudaEvent_t> probe_cap;    // the events recorded at capture
  };
  using GraphKey = std::tuple<int, int, int, int, int>;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> cap_probes;  // filled while capturing
  std::map<GraphKey, GraphEntry> graphs;
  std::map<GraphKey, int> graph_seen;
  int use_graph = 1;        // option "graph": 0 off, 1 capture on a shape's second run, 2 on its first
  bool capturing = false;   // inside a capture: grids sized for the bucket's maximum row counts
  long long graph_replays = 0;
  void drop_graphs() {
    for (auto& kv : graphs) {
      cudaGraphExecDestroy(kv.second.exec);
      cudaGraphDestroy(kv.second.graph);
      for (cudaEvent_t ev : kv.second.probe_cap) cudaEventDestroy(ev);
    }
    graphs.clear();
    graph_seen.clear();
  }
  bool graph_ok(bool dp) const {
    return use_graph && !dp && !g_tl.on && ncu_class < 0 && stop_after == 0 && trace_layer < 0;
  }
  // grid for the embedding-row kernels: the batch's count (eager) or the
  // bucket's maximum (captured; the kernels read the count from the scalars)
  int rows_grid(int t) const { return (capturing || seg_dev) ? nrows_max[t] : nuniq[t]; }
  // host view of a table's unique rows (device-segment mode: from the staged ids)
  void host_segments(int t) {
    if (!seg_dev || seg_host_ok[t]) return;
    std::vector<int> u = seg_ids_h[t];
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    uniq_h[t] = u;
    nuniq[t] = (int)u.size();
    seg_host_ok[t] = true;
  }
  int host_rows(int t) {
    host_segments(t);
    return (int)uniq_h[t].size();
  }
  void launch_segments() {
    const long long NS = (long long)S * B, NT = (long long)T * B;
    SegJob j[2];
    for (int t = 0; t < 2; ++t) {
      j[t].off = seg_off_d[t]; j[t].pos = seg_pos_d[t]; j[t].uq = uniq_d[t]; j[t].nrows = &scal_d->nrows[t];
      j[t].ids1 = nullptr; j[t].n1 = 0;
    }
    j[0].ids0 = src_ids_d; j[0].n0 = (int)NS; j[0].pos_base = 0;
    if (cfg.shared_embeddings) { j[0].ids1 = tgt_in_d; j[0].n1 = (int)NT; }
    j[1].ids0 = tgt_in_d; j[1].n0 = (int)NT; j[1].pos_base = (int)NS;
    int bits = 0;
    while (bits < 31 && ((long long)(V - 1) >> bits)) ++bits;
    const int nmax = (int)std::max<long long>(j[0].n0 + j[0].n1, n_tables > 1 ? j[1].n0 : 0);
    static bool attr = false;
    if (!attr) {
      CMT_CUDA(cudaFuncSetAttribute(segments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)seg_smem(SEG_MAX_N)));
      attr = true;
    }
    ncu_begin(14);
    segments_kernel<<<n_tables, SEG_THREADS, seg_smem(nmax), st>>>(j[0], j[1], bits);
    ncu_end();
    CMT_LAUNCHED(); tl_mark(st, "segments_kernel");
  }
  const int* rows_dev(int t) const { return &scal_d->nrows[t]; }

  void run(const cmt_step_args& a, cmt_step_result* res) {
    if (!staged) throw Error(CMT_ERR_INTERNAL, "no batch staged");
    const bool dp = comm != nullptr;  // (a 1-rank communicator exercises the same path)
    const bool infer = (a.flags & CMT_FLAG_INFER) != 0;  // dev_entropy pass (training.py:162-182)
    const bool drop = cfg.dropout > 0.0 && !infer;        // INFER mode: dropout is the identity
    Pcg pcg{a.pcg_state_hi, a.pcg_state_lo, a.pcg_inc_hi, a.pcg_inc_lo};
    if (drop) ensure_jump(pcg);  // before any side-stream dropout reads the table
    double ntok = a.global_ntok > 0 ? a.global_ntok : ntok_local;
    float inv_ntok = ntok > 0 ? (float)(1.0 / (double)(float)ntok) : 0.f;
    StepScalars sv;
    sv.pcg = pcg;
    sv.lr = a.lr;
    sv.clip = a.clip_norm;
    sv.eps = (float)a.epsilon;
    sv.inv_ntok = inv_ntok;
    sv.nrows[0] = nuniq[0];
    sv.nrows[1] = nuniq[1];
    set_scalars_kernel<<<1, 1, 0, st>>>(sv, scal_d);
    CMT_LAUNCHED(); tl_mark(st, "set_scalars_kernel");
    last_infer = infer;
    last_ntok = ntok;
    unsigned long long draws = 0;
    if (graph_ok(dp)) {
      const GraphKey key{S, T, B, a.flags & (CMT_FLAG_INFER | CMT_FLAG_NO_UPDATE), time_dominant};
      auto it = graphs.find(key);
      if (it == graphs.end() && ++graph_seen[key] >= (use_graph >= 2 ? 1 : 2)) {
        if (graphs.size() >= 16) drop_graphs();  // many shapes (e.g. beam-search encodes): start over
        const unsigned long long l0 = g_launches;
        cudaGraph_t g = nullptr;
        capturing = true;
        cap_probes.clear();
        CMT_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        try {
          draws = step_body(a, dp);
        } catch (...) {
          cudaStreamEndCapture(st, &g);
          if (g) cudaGraphDestroy(g);
          capturing = false;
          throw;
        }
        capturing = false;
        CMT_CUDA(cudaStreamEndCapture(st, &g));
        GraphEntry ge;
        ge.graph = g;
        cudaError_t err = cudaGraphInstantiate(&ge.exec, g, 0);
        if (err != cudaSuccess) cudaGraphDestroy(g);
        CMT_CUDA(err);
        // probes: each replay records fresh events into the captured record nodes
        for (size_t i = 0; i < cap_probes.size(); ++i) {
          ge.probe_cls.push_back(cap_probes[i].first);
          ge.probe_cap.push_back(cap_probes[i].second.first);
          ge.probe_cap.push_back(cap_probes[i].second.second);
        }
        if (!cap_probes.empty()) {
          size_t n = 0;
          CMT_CUDA(cudaGraphGetNodes(g, nullptr, &n));
          std::vector<cudaGraphNode_t> nodes(n);
          CMT_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
          for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            CMT_CUDA(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeEventRecord) continue;
            cudaEvent_t ev;
            CMT_CUDA(cudaGraphEventRecordNodeGetEvent(nd, &ev));
            for (size_t i = 0; i < cap_probes.size(); ++i) {
              if (ev == cap_probes[i].second.first) ge.probe_nodes.push_back({nd, (int)i, true});
              if (ev == cap_probes[i].second.second) ge.probe_nodes.push_back({nd, (int)i, false});
            }
          }
          if (ge.probe_nodes.size() != 2 * cap_probes.size())
            throw Error(CMT_ERR_INTERNAL, "captured probe events not found in the step graph");
        }
        cap_probes.clear();
        ge.draws = draws;
        ge.kernels = g_launches - l0;
        g_launches = l0;
        it = graphs.emplace(key, ge).first;
      }
      if (it != graphs.end()) {
        GraphEntry& ge = it->second;
        if (!ge.probe_cls.empty()) {
          std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs(ge.probe_cls.size());
          for (auto& pr : evs) {
            pr.first = pooled_event();
            pr.second = pooled_event();
          }
          for (const ProbeNode& pn : ge.probe_nodes)
            CMT_CUDA(cudaGraphExecEventRecordNodeSetEvent(ge.exec, pn.node,
                                                          pn.begin ? evs[pn.pair].first : evs[pn.pair].second));
          for (size_t i = 0; i < evs.size(); ++i) probe_ev[ge.probe_cls[i]].push_back(evs[i]);
        }
        CMT_CUDA(cudaGraphLaunch(it->second.exec, st));
        g_launches += it->second.kernels;
        ++graph_replays;
        draws = it->second.draws;
      } else {
        draws = step_body(a, dp);
      }
    } else {
      draws = step_body(a, dp);
    }
    last_draws = draws;
    if (res) {
      res->draws = draws;
      res->status = CMT_OK;
      if (!(a.flags & CMT_FLAG_ASYNC)) wait(res);
    }
  }

  // the step's launches (captured into a graph or issued eagerly); returns the draws
  unsigned long long step_body(const cmt_step_args& a, bool dp) {
    emb_sent[0] = emb_sent[1] = false;
    const long long NS = (long long)S * B, NT = (long long)T * B, BH = (long long)B * H;
    const bool infer = (a.flags & CMT_FLAG_INFER) != 0;
    const bool drop = cfg.dropout > 0.0 && !infer;
    const Pcg* pcg = &scal_d->pcg;
    bool seg_pending = seg_dev && !infer;  // the embedding segments, before the backward needs them
    CMT_CUDA(cudaMemsetAsync(out_d, 0, sizeof(StepOut), st));
    // every recurrent launch of the step owns one flag region (forward layer l:
    // region l, BPTT: region nlayers + l): one memset instead of one per launch
    CMT_CUDA(cudaMemsetAsync(flags, 0, flag_words() * 4, st));
    if (g_tl.on) {
      hold_kernel<<<1, 1, 0, st>>>(20000000ull);  // 20 ms: the host enqueues the step meanwhile
      CMT_LAUNCHED();
    }
    tl_mark(st, "<start>");

    // ===== forward =====
    gather(0, src_ids_d, (int)NS, Xs);
    gather(tgt_table(), tgt_in_d, (int)NT, Xt);
    for (int l : {0, 1}) {  // zero initial states of the encoder scans
      ScanViews v = views(l, l == 1);
      CMT_CUDA(cudaMemsetAsync((char*)v.hprev + (size_t)(l == 1 ? (S - 1) : 0) * BH * asz, 0, BH * asz, st));
      CMT_CUDA(cudaMemsetAsync((float*)v.cprev + (size_t)(l == 1 ? (S - 1) : 0) * BH, 0, BH * 4, st));
    }
    // dropout draw bases in the reference's draw order: encoder
    // sites k=2..L, then decoder sites k=2..L, then H_o
    auto enc_base = [&](int k) { return (unsigned long long)(k - 2) * NS * H; };
    auto dec_base = [&](int k) { return (unsigned long long)(L - 1) * NS * H + (unsigned long long)(k - 2) * NT * H; };
    unsigned long long draw = drop ? (unsigned long long)(L - 1) * (NS + NT) * H : 0;
    // masks ahead of the sites (bf16, paired TMEM scans, side stream available):
    // site ids: encoder k -> k, decoder k -> L + k, H_o -> 2L + 1
    const bool ahead = drop && mask_ahead && bf && use_dual_fwd() && dual_tm();
    mask_queue.clear();
    auto queue_mask = [&](int id, uint8_t* keep, long long n, unsigned long long base) {
      if (ahead) mask_queue.push_back({id, keep, (int)n, base});
    };
    auto dropout_site = [&](const void* in, void* out, uint8_t* keep, long long n, unsigned long long base) {
      if (bf) launch_dropout<bf16, bf16>(in, out, keep, (int)n, base, pcg);
      else launch_dropout<float, float>(in, out, keep, (int)n, base, pcg);
    };
    // decoder layer k starts from encoder layer k's final state (model.py:292-305);
    // l1.bwd's final sits in slot 0, deep layers' in slot S
    auto dec_init = [&](int k) {
      int el = (k == 1) ? 1 : k;
      size_t fslot = (k == 1) ? 0 : (size_t)S;
      copy_act((char*)lw[el].yext + fslot * BH * asz, H, lw[L + k].yext, H, B, H);
      CMT_CUDA(cudaMemcpyAsync(lw[L + k].cext, lw[el].cext + fslot * BH, BH * 4, cudaMemcpyDeviceToDevice, st));
    };
    // input of decoder layer k (k >= 2: dropout of layer k-1's output)
    auto dec_input = [&](int k) -> const void* {
      if (k == 1) return Xt;
      const void* prev = views(L + k - 1, false).ybase;
      if (!drop) { drop_dec[k] = const_cast<void*>(prev); return prev; }
      if (ahead) apply_dropout<bf16, bf16>(L + k, prev, nullptr, keep_dec[k], drop_dec[k], NT * H);
      else dropout_site(prev, drop_dec[k], keep_dec[k], NT, dec_base(k));
      return drop_dec[k];
    };
    auto enc_input = [&](int k, const void* cur) -> const void* {
      if (!drop) { drop_enc[k] = const_cast<void*>(cur); return cur; }
      if (ahead) apply_dropout<bf16, bf16>(k, cur, nullptr, keep_enc[k], drop_enc[k], NS * H);
      else dropout_site(cur, drop_enc[k], keep_enc[k], NS, enc_base(k));
      return drop_enc[k];
    };
    // enc.l2's input: dropout(y_f + y_b) in one pass (the sum is not stored)
    auto enc_input_l1sum = [&]() -> const void* {
      ScanViews f = views(0, false), r = views(1, true);
      if (ahead) apply_dropout<bf16, bf16>(2, f.ybase, r.ybase, keep_enc[2], drop_enc[2], NS * H);
      else if (bf) launch_dropout<bf16, bf16>(f.ybase, drop_enc[2], keep_enc[2], (int)NS, enc_base(2), pcg, r.ybase);
      else launch_dropout<float, float>(f.ybase, drop_enc[2], keep_enc[2], (int)NS, enc_base(2), pcg, r.ybase);
      return drop_enc[2];
    };
    auto add_top = [&]() {
      ScanViews f = views(0, false), r = views(1, true);
      if (bf) add2_kernel<bf16><<<grid_for(NS * H), 256, 0, st>>>((const bf16*)f.ybase, (const bf16*)r.ybase, (bf16*)top, NS * H);
      else add2_kernel<float><<<grid_for(NS * H), 256, 0, st>>>((const float*)f.ybase, (const float*)r.ybase, (float*)top, NS * H);
      CMT_LAUNCHED(); tl_mark(st, "add2_kernel");
    };
    auto zero_enc_state = [&](int k) {
      CMT_CUDA(cudaMemsetAsync(lw[k].yext, 0, BH * asz, st));
      CMT_CUDA(cudaMemsetAsync(lw[k].cext, 0, BH * 4, st));
    };
    if (use_dual_fwd()) {
      // two independent scans per launch: (e1f, e1b), (e2, d1), ..., (eL, d(L-1)), then dL
      FwdScan a{0, Xs, E, S, false, src_mask_d, ux}, b{1, Xs, E, S, true, src_mask_d, ux2};
      if (use_overlap()) {
        fork();
        fwd_prep(a);
        on_side_stream([&]() { fwd_prep(b); });
        join();
      } else {
        fwd_prep(a);
        fwd_prep(b);
      }
      // dec.l1's input projection depends only on the target embeddings: on the
      // side stream, capped to the SMs the paired enc.l1 scans leave idle, it
      // runs beside them instead of in level 2
      const int idle = g_num_sms - 2 * (dual_tm() ? tm::Fwd<64>::ctas(H, B) : mc::Fwd<128>::ctas(H, B));
      const bool dec1_early = early_dec1 && use_overlap() && L >= 2 && idle >= 8;
      FwdScan d1{L + 1, Xt, E, T, false, nullptr, ux3};
      if (dec1_early) fork();
      if (L >= 2) queue_mask(2, keep_enc[2], NS, enc_base(2));  // enc.l2's input, beside the enc.l1 scans
      fwd_pair(a, b);
      if (dec1_early) {
        on_side_stream([&]() {
          g_grid_cap = idle;
          fwd_prep(d1);
          g_grid_cap = 0;
          if (seg_pending) {  // two CTAs on the SMs the enc.l1 scans leave idle
            launch_segments();
            seg_pending = false;
          }
        });
      }
      // with dropout the summed top is only the input of enc.l2's dropout site:
      // the sum is formed inside that dropout kernel (no separate add pass)
      const bool fused_top = drop && L >= 2;
      if (!fused_top) add_top();
      const void* cur = top;
      for (int k = 2; k <= L; ++k) {
        // the two scans' inputs (dropout, initial state, input projection) are
        // independent: the decoder side is issued on the side stream
        const bool ov = use_overlap();
        if (ov) fork();
        const void* in = (k == 2 && fused_top) ? enc_input_l1sum() : enc_input(k, cur);
        zero_enc_state(k);
        FwdScan e{k, in, H, S, false, src_mask_d, ux};
        fwd_prep(e);
        const void* xd = nullptr;
        auto dec_side = [&]() {
          xd = dec_input(k - 1);
          dec_init(k - 1);
        };
        if (ov) on_side_stream(dec_side);
        else dec_side();
        FwdScan d{L + k - 1, xd, k - 1 == 1 ? E : H, T, false, nullptr, ux2};
        if (k == 2 && dec1_early) {
          d = d1;  // projected beside the enc.l1 scans (joined here)
          join();
        } else if (ov) {
          on_side_stream([&]() { fwd_prep(d); });
          join();
        } else {
          fwd_prep(d);
        }
        if (k + 1 <= L) queue_mask(k + 1, keep_enc[k + 1], NS, enc_base(k + 1));
        queue_mask(L + k, keep_dec[k], NT, dec_base(k));  // dec.lk's input, applied at the next level
        fwd_pair(e, d);
        cur = views(k, false).ybase;
      }
      const void* xd = dec_input(L);
      dec_init(L);
      queue_mask(2 * L + 1, keep_o, NT, draw);  // H_o, beside the dec.lL scan
      scan_fwd(2 * L, xd, L == 1 ? E : H, T, false, nullptr);
      flush_masks(0);  // (a scan path without a persistent launch: generate them here)
    } else {
      scan_fwd(0, Xs, E, S, false, src_mask_d);
      scan_fwd(1, Xs, E, S, true, src_mask_d);
      add_top();
      const void* cur = top;
      for (int k = 2; k <= L; ++k) {
        const void* in = enc_input(k, cur);
        zero_enc_state(k);
        scan_fwd(k, in, H, S, false, src_mask_d);
        cur = views(k, false).ybase;
      }
      for (int k = 1; k <= L; ++k) {
        const void* x = dec_input(k);
        dec_init(k);
        scan_fwd(L + k, x, k == 1 ? E : H, T, false, nullptr);
      }
    }
    if (seg_pending) {
      launch_segments();
      seg_pending = false;
    }
    const void* Hs = (L == 1) ? top : views(L, false).ybase;
    const void* Ht = views(2 * L, false).ybase;
    // attention (attention.py:146-173)
    copy_act(Ht, H, (char*)cst_att + (size_t)H * asz, 2LL * H, (int)NT, H);
    gemm((int)NT, H, H, Mat{Ht, H, 0}, Mat{wv(off_wa), H, 1}, store(u_att, H, true));
    if (att_tc_ok()) {
      // tcgen05: scores = U Hs^T, masked softmax, C_s = alpha Hs (attention_tc.cuh)
      ncu_begin(9);
      att_tc_ts(u_att, att_dsc);
      ncu_end();
      att_softmax_fwd_kernel<<<ceil_div(B * T, 8), 256, 0, st>>>(att_dsc, src_mask_d, S, T, B, s8(), alpha, att_a16,
                                                                 status_d);
      CMT_LAUNCHED(); tl_mark(st, "attn_tc_softmax");
      att_tc_th(att_a16, cst_att, (long long)B * 2 * H, 2LL * H, 1);
    } else if (S <= att2::MAXL && T <= att2::MAXL && att_split == 2) {
      const int nsp = att::nslices(H), tt = att2::tiles(T), ts = att2::tiles(S);
      dim3 gs(B, nsp, tt * ts), gc(B, ceil_div(H, att::HC), tt);
      if (bf) attn2_scores_part<bf16, bf16><<<gs, att::THREADS, 0, st>>>((const bf16*)u_att, H, (const bf16*)Hs, S, T, B,
                                                                        H, att_part);
      else attn2_scores_part<float, float><<<gs, att::THREADS, 0, st>>>((const float*)u_att, H, (const float*)Hs, S, T, B,
                                                                        H, att_part);
      CMT_LAUNCHED(); tl_mark(st, "attn2_scores_part");
      attn2_rows<<<B, att::THREADS, 0, st>>>(att_part, nsp, src_mask_d, S, T, B, alpha, nullptr, 0, status_d);
      CMT_LAUNCHED(); tl_mark(st, "attn2_rows");
      const size_t smem = sizeof(float) * 2 * ts * att2::P * att::LD;
      if (bf) {
        CMT_CUDA(cudaFuncSetAttribute(attn2_ws_hs<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attn2_ws_hs<bf16><<<gc, att::THREADS, smem, st>>>((const bf16*)Hs, alpha, S, T, B, H, (bf16*)cst_att, 2LL * H);
      } else {
        CMT_CUDA(cudaFuncSetAttribute(attn2_ws_hs<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attn2_ws_hs<float><<<gc, att::THREADS, smem, st>>>((const float*)Hs, alpha, S, T, B, H, (float*)cst_att, 2LL * H);
      }
      CMT_LAUNCHED(); tl_mark(st, "attn2_context");
      CMT_CUDA(cudaGetLastError());
    } else if (S <= att::P && T <= att::P && att_split) {
      const int nsp = att::nslices(H);
      dim3 gs(B, nsp), gc(B, ceil_div(H, att::HC));
      if (bf) attn_scores_part<bf16, bf16><<<gs, att::THREADS, 0, st>>>((const bf16*)u_att, H, (const bf16*)Hs, S, T, B, H,
                                                                       att_part);
      else attn_scores_part<float, float><<<gs, att::THREADS, 0, st>>>((const float*)u_att, H, (const float*)Hs, S, T, B,
                                                                       H, att_part);
      CMT_LAUNCHED(); tl_mark(st, "attn_scores_part");
      attn_softmax_fwd<<<B, att::THREADS, 0, st>>>(att_part, nsp, src_mask_d, S, T, B, alpha, status_d);
      CMT_LAUNCHED(); tl_mark(st, "attn_softmax_fwd");
      if (bf) attn_context<bf16><<<gc, att::THREADS, 0, st>>>((const bf16*)Hs, alpha, S, T, B, H, (bf16*)cst_att, 2LL * H);
      else attn_context<float><<<gc, att::THREADS, 0, st>>>((const float*)Hs, alpha, S, T, B, H, (float*)cst_att, 2LL * H);
      CMT_LAUNCHED(); tl_mark(st, "attn_context");
      CMT_CUDA(cudaGetLastError());
    } else if (S <= att::P && T <= att::P) {
      const size_t smem = att::fwd_smem();
      if (bf) {
        CMT_CUDA(cudaFuncSetAttribute(attn_fwd_tiled<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attn_fwd_tiled<bf16><<<B, att::THREADS, smem, st>>>((const bf16*)Hs, (const bf16*)u_att, src_mask_d, S, T, B, H,
                                                            alpha, (bf16*)cst_att, 2LL * H, status_d);
      } else {
        CMT_CUDA(cudaFuncSetAttribute(attn_fwd_tiled<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attn_fwd_tiled<float><<<B, att::THREADS, smem, st>>>((const float*)Hs, (const float*)u_att, src_mask_d, S, T, B,
                                                             H, alpha, (float*)cst_att, 2LL * H, status_d);
      }
      CMT_LAUNCHED(); tl_mark(st, "attn_fwd_tiled");
      CMT_CUDA(cudaGetLastError());
    } else {
      size_t smem = attn_fwd_smem(S, T);
      if (bf) {
        cudaFuncSetAttribute(attn_fwd_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attn_fwd_kernel<bf16><<<B, ATT_THREADS, smem, st>>>((const bf16*)Hs, (const bf16*)u_att, src_mask_d, S, T, B, H,
                                                              alpha, (bf16*)cst_att, 2LL * H, status_d);
      } else {
        cudaFuncSetAttribute(attn_fwd_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attn_fwd_kernel<float><<<B, ATT_THREADS, smem, st>>>((const float*)Hs, (const float*)u_att, src_mask_d, S, T, B,
                                                               H, alpha, (float*)cst_att, 2LL * H, status_d);
      }
      CMT_LAUNCHED(); tl_mark(st, "attn_fwd_kernel");
      CMT_CUDA(cudaGetLastError());
    }
    {
      EpiStore e = store(ho, H, false);
      e.act = 1;
      gemm((int)NT, H, 2 * H, Mat{cst_att, 2LL * H, 0}, Mat{wv(off_wc), H, 1}, e);
    }
    const void* hin = ho;
    if (drop) {
      if (ahead) apply_dropout<float, bf16>(2 * L + 1, ho, nullptr, keep_o, hod, NT * H);
      else if (bf) launch_dropout<float, bf16>(ho, hod, keep_o, (int)NT, draw, pcg);
      else launch_dropout<float, float>(ho, hod, keep_o, (int)NT, draw, pcg);
      draw += (unsigned long long)NT * H;
      hin = hod;
    } else {
      if (bf) {
        copy2d_kernel<float, bf16><<<grid_for(NT * H), 256, 0, st>>>(ho, H, (bf16*)hod, H, (int)NT, H);
        CMT_LAUNCHED(); tl_mark(st, "copy2d_kernel");
      } else {
        CMT_CUDA(cudaMemcpyAsync(hod, ho, NT * H * 4, cudaMemcpyDeviceToDevice, st));
      }
      hin = hod;
    }
    {
      EpiStore e = store(Y, V, true);
      e.bias = dw + off_bo;
      e.act = cfg.output_tanh ? 1 : 0;
      cudaEvent_t e0 = probe_begin(0);
      gemm((int)NT, V, H, Mat{hin, H, 0}, Mat{wv(off_wo), V, 1}, e);
      probe_end(0, e0);
    }
    if (stop_after == 1) { CMT_CUDA(cudaStreamSynchronize(st)); return 0; }
    // fused log-softmax + smoothed CE + grad (training.py:96-120, tensor.py:146-151)
    const bool fused_ce = use_ce2() && cepart;
    if (fused_ce) {
      ncu_begin(6);
      ce_stats_kernel<<<(int)NT, CES_THREADS, 0, st>>>((const bf16*)Y, V, tgt_out_d, tgt_mask_d, scal_d,
                                                       cfg.output_tanh, losstok, status_d, cerow);
      ncu_end();
      CMT_LAUNCHED(); tl_mark(st, "ce_stats_kernel");
      const int chunks = (int)ceil_div(NT, CEG_ROWS);
      ncu_begin(7);
      ce_grad_kernel<<<dim3(ceil_div(V, CEG_COLS), chunks), CEG_THREADS, 0, st>>>((bf16*)Y, V, (int)NT, tgt_out_d,
                                                                                  cerow, scal_d,
                                                                                  cfg.output_tanh, cepart);
      ncu_end();
      CMT_LAUNCHED(); tl_mark(st, "ce_grad_kernel");
      colsum_final_kernel<<<ceil_div(V, 256), 256, 0, st>>>(cepart, chunks, V, dg + off_bo);
      CMT_LAUNCHED(); tl_mark(st, "colsum_final_kernel");
    } else {
      if (bf) ce_kernel<bf16><<<(int)NT, CE_THREADS, 0, st>>>((bf16*)Y, V, tgt_out_d, tgt_mask_d, scal_d,
                                                              cfg.output_tanh, losstok, status_d);
      else ce_kernel<float><<<(int)NT, CE_THREADS, 0, st>>>((float*)Y, V, tgt_out_d, tgt_mask_d, scal_d,
                                                            cfg.output_tanh, losstok, status_d);
      CMT_LAUNCHED(); tl_mark(st, "ce_kernel");
    }
    sum_to_double_kernel<<<1, 1024, 0, st>>>(losstok, (int)NT, losssum_d);
    CMT_LAUNCHED(); tl_mark(st, "sum_to_double_kernel");

    if (stop_after == 2) { CMT_CUDA(cudaStreamSynchronize(st)); return 0; }
    if (infer) {  // forward only: loss sum and token count, no backward, no update, no draws
      CMT_CUDA(cudaGetLastError());
      CMT_CUDA(cudaMemcpyAsync(out_h, out_d, sizeof(StepOut), cudaMemcpyDeviceToHost, st));
      return 0;
    }
    // ===== backward =====
    // output projection (layers.py:64-73): dW_o, db_o, dH_o (+ dropout bwd + tanh' of H_o)
    // dW_o only feeds the update: on the side stream it overlaps dH_o and the
    // attention backward (joined before the BPTT scans)
    const bool ov_wo = use_overlap();
    ar_buckets = comm != nullptr && ar_overlap && ov_wo;
    ar_done.assign(layers.size() + 2, 0);
    n_ev_ar = 0;
    if (ov_wo) {
      fork();
      on_side_stream([&]() {
        ncu_begin(11);
        gemm(H, V, (int)NT, Mat{hin, H, 1}, Mat{Y, V, 1}, store(dg + off_wo, V, false));
        ncu_end();
        if (!fused_ce) colsum(Y, true, NT, V, dg + off_bo);
        allreduce_region((int)layers.size() + 1);
      });
    } else {
      gemm(H, V, (int)NT, Mat{hin, H, 1}, Mat{Y, V, 1}, store(dg + off_wo, V, false));
      if (!fused_ce) colsum(Y, true, NT, V, dg + off_bo);
    }
    {
      // dH_o = dY W_o^T with the dropout mask and tanh' of H_o applied (linear, so
      // they may act per K slice).  bf16 mode: K = V is long and the 100 output
      // tiles leave pairs idle, so the product is split-K into an fp32 scratch
      // and converted to the bf16 activation afterwards.
      const bool via32 = bf && dho32 && pick_ks((int)NT, H, V, 256, 2) != 1;
      EpiStore e = via32 ? store(dho32, H, false) : store(dhpre, H, true);
      if (drop) { e.dmask = keep_o; e.ld_dmask = H; e.dscale = 1.0f / (float)(1.0 - cfg.dropout); }
      e.tgrad_y = ho; e.ld_tgrad = H;
      gemm((int)NT, H, V, Mat{Y, V, 0}, Mat{wv(off_wo), V, 0}, e);
      if (via32) {
        copy2d_kernel<float, bf16><<<grid_for(NT * H), 256, 0, st>>>(dho32, H, (bf16*)dhpre, H, (int)NT, H);
        CMT_LAUNCHED(); tl_mark(st, "copy2d_kernel");
      }
    }
    // W_c (attention.py:171)
    gemm(2 * H, H, (int)NT, Mat{cst_att, 2LL * H, 1}, Mat{dhpre, H, 1}, store(dg + off_wc, H, false));
    gemm((int)NT, 2 * H, H, Mat{dhpre, H, 0}, Mat{wv(off_wc), H, 0}, store(dcst, 2LL * H, false));
    // attention core backward
    float* dHs = (L == 1) ? dtop : lw[L].dy;
    if (att_tc_ok()) {
      // tcgen05 (attention_tc.cuh): dalpha = dC Hs^T, softmax backward,
      // dU = dsc Hs, dHs = alpha^T dC + dsc^T U (every row of dHs written)
      copy2d_kernel<float, bf16><<<grid_for(NT * H), 256, 0, st>>>(dcst, 2LL * H, att_dc16, H, (int)NT, H);
      CMT_LAUNCHED(); tl_mark(st, "attn_tc_dc16");
      att_tc_ts(att_dc16, att_dsc);
      att_softmax_bwd_kernel<<<ceil_div(B * T, 8), 256, 0, st>>>(alpha, att_dsc, S, T, B, s8(), att_d16);
      CMT_LAUNCHED(); tl_mark(st, "attn_tc_softmax_bwd");
      att_tc_th(att_d16, du_att, (long long)B * H, H, 1);
      const BatOp aT{att_a16, S, T, (long long)T * s8() * 2, s8() * 2LL, 2},
          dT{att_d16, S, T, (long long)T * s8() * 2, s8() * 2LL, 2},
          dcb{att_dc16, H, T, H * 2LL, (long long)B * H * 2, 1}, ub{u_att, H, T, H * 2LL, (long long)B * H * 2, 1};
      bat_gemm<256, 1, 1>(S, H, T, B, aT, dcb, BatStore{dHs, (long long)B * H, H, 0, 0});
      bat_gemm<256, 1, 1>(S, H, T, B, dT, ub, BatStore{dHs, (long long)B * H, H, 0, 1});
    } else {
    CMT_CUDA(cudaMemsetAsync(dHs, 0, NS * H * 4, st));
    if (S <= att2::MAXL && T <= att2::MAXL && att_split == 2) {
      const int nsp = att::nslices(H), tt = att2::tiles(T), ts = att2::tiles(S);
      dim3 gs(B, nsp, tt * ts), gt(B, ceil_div(H, att::HC), tt), gsd(B, ceil_div(H, att::HC), ts);
      if (bf) attn2_scores_part<float, bf16><<<gs, att::THREADS, 0, st>>>(dcst, 2LL * H, (const bf16*)Hs, S, T, B, H,
                                                                         att_part);
      else attn2_scores_part<float, float><<<gs, att::THREADS, 0, st>>>(dcst, 2LL * H, (const float*)Hs, S, T, B, H,
                                                                         att_part);
      CMT_LAUNCHED(); tl_mark(st, "attn2_scores_part");
      attn2_rows<<<B, att::THREADS, 0, st>>>(att_part, nsp, src_mask_d, S, T, B, alpha, att_dsc, 1, status_d);
      CMT_LAUNCHED(); tl_mark(st, "attn2_rows");
      const size_t smem_h = sizeof(float) * 4 * tt * att2::P * att::LD;
      const size_t smem_u = sizeof(float) * 2 * ts * att2::P * att::LD;
      if (bf) {
        CMT_CUDA(cudaFuncSetAttribute(attn2_dhs<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_h));
        attn2_dhs<bf16><<<gsd, att::THREADS, smem_h, st>>>((const bf16*)u_att, alpha, att_dsc, dcst, 2LL * H, S, T, B, H,
                                                           dHs);
        CMT_LAUNCHED(); tl_mark(st, "attn2_dhs");
        CMT_CUDA(cudaFuncSetAttribute(attn2_ws_hs<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_u));
        attn2_ws_hs<bf16><<<gt, att::THREADS, smem_u, st>>>((const bf16*)Hs, att_dsc, S, T, B, H, (bf16*)du_att, H);
      } else {
        CMT_CUDA(cudaFuncSetAttribute(attn2_dhs<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_h));
        attn2_dhs<float><<<gsd, att::THREADS, smem_h, st>>>((const float*)u_att, alpha, att_dsc, dcst, 2LL * H, S, T, B,
                                                            H, dHs);
        CMT_LAUNCHED(); tl_mark(st, "attn2_dhs");
        CMT_CUDA(cudaFuncSetAttribute(attn2_ws_hs<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_u));
        attn2_ws_hs<float><<<gt, att::THREADS, smem_u, st>>>((const float*)Hs, att_dsc, S, T, B, H, (float*)du_att, H);
      }
      CMT_LAUNCHED(); tl_mark(st, "attn2_du");
      CMT_CUDA(cudaGetLastError());
    } else if (S <= att::P && T <= att::P && att_split) {
      const int nsp = att::nslices(H);
      dim3 gs(B, nsp), gc(B, ceil_div(H, att::HC));
      if (bf) attn_scores_part<float, bf16><<<gs, att::THREADS, 0, st>>>(dcst, 2LL * H, (const bf16*)Hs, S, T, B, H, att_part);
      else attn_scores_part<float, float><<<gs, att::THREADS, 0, st>>>(dcst, 2LL * H, (const float*)Hs, S, T, B, H, att_part);
      CMT_LAUNCHED(); tl_mark(st, "attn_scores_part");
      attn_dscores<<<B, att::THREADS, 0, st>>>(att_part, nsp, alpha, S, T, att_dsc);
      CMT_LAUNCHED(); tl_mark(st, "attn_dscores");
      const size_t smem = sizeof(float) * 6 * att::P * att::LD;
      if (bf) {
        CMT_CUDA(cudaFuncSetAttribute(attn_bwd_chunk<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attn_bwd_chunk<bf16><<<gc, att::THREADS, smem, st>>>((const bf16*)Hs, (const bf16*)u_att, alpha, att_dsc, dcst,
                                                             2LL * H, S, T, B, H, dHs, (bf16*)du_att);
      } else {
        CMT_CUDA(cudaFuncSetAttribute(attn_bwd_chunk<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attn_bwd_chunk<float><<<gc, att::THREADS, smem, st>>>((const float*)Hs, (const float*)u_att, alpha, att_dsc, dcst,
                                                              2LL * H, S, T, B, H, dHs, (float*)du_att);
      }
      CMT_LAUNCHED(); tl_mark(st, "attn_bwd_chunk");
      CMT_CUDA(cudaGetLastError());
    } else if (S <= att::P && T <= att::P) {
      const size_t smem = att::bwd_smem();
      if (bf) {
        CMT_CUDA(cudaFuncSetAttribute(attn_bwd_tiled<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attn_bwd_tiled<bf16><<<B, att::THREADS, smem, st>>>((const bf16*)Hs, (const bf16*)u_att, alpha, dcst, 2LL * H, S, T,
                                                            B, H, dHs, (bf16*)du_att);
      } else {
        CMT_CUDA(cudaFuncSetAttribute(attn_bwd_tiled<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attn_bwd_tiled<float><<<B, att::THREADS, smem, st>>>((const float*)Hs, (const float*)u_att, alpha, dcst, 2LL * H, S,
                                                             T, B, H, dHs, (float*)du_att);
      }
      CMT_LAUNCHED(); tl_mark(st, "attn_bwd_tiled");
      CMT_CUDA(cudaGetLastError());
    } else {
      size_t smem = attn_bwd_smem(S, T);
      if (bf) {
        cudaFuncSetAttribute(attn_bwd_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attn_bwd_kernel<bf16><<<B, ATT_THREADS, smem, st>>>((const bf16*)Hs, (const bf16*)u_att, alpha, dcst, 2LL * H, S, T,
                                                              B, H, dHs, (bf16*)du_att);
      } else {
        cudaFuncSetAttribute(attn_bwd_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attn_bwd_kernel<float><<<B, ATT_THREADS, smem, st>>>((const float*)Hs, (const float*)u_att, alpha, dcst, 2LL * H, S,
                                                               T, B, H, dHs, (float*)du_att);
      }
      CMT_LAUNCHED(); tl_mark(st, "attn_bwd_kernel");
      CMT_CUDA(cudaGetLastError());
    }
    }
    // W_a (attention.py:166): dW_a and dH_t = du W_a^T + dC_st[:, H:]
    gemm(H, H, (int)NT, Mat{Ht, H, 1}, Mat{du_att, H, 1}, store(dg + off_wa, H, false));
    {
      EpiStore e = store(lw[2 * L].dy, H, false);
      e.add = dcst + H; e.ld_add = 2LL * H;
      gemm((int)NT, H, H, Mat{du_att, H, 0}, Mat{wv(off_wa), H, 0}, e);
    }
    allreduce_region((int)layers.size());
    if (ov_wo) join();
    // decoder BPTT, top layer first (graph.py:112-115); init-state grads -> encoder finals
    auto dec_scan = [&](int k, void* dub) {
      BwdScan f;
      f.l = L + k; f.X = (k == 1) ? Xt : drop_dec[k]; f.din = (k == 1) ? E : H; f.steps = T; f.reverse = false;
      f.mask = nullptr; f.dy = lw[L + k].dy; f.dh_final = nullptr; f.dc_final = nullptr;
      f.dh0 = fin_dh[k]; f.dc0 = fin_dc[k];
      f.dX = (k == 1) ? dXemb + NS * E : lw[L + k - 1].dy; f.dx_beta = 0;
      f.dx_keep = (k > 1 && drop) ? keep_dec[k] : nullptr; f.dUb = dub;
      return f;
    };
    auto enc_scan = [&](int k, void* dub) {  // k >= 2
      BwdScan f;
      f.l = k; f.X = drop_enc[k]; f.din = H; f.steps = S; f.reverse = false; f.mask = src_mask_d; f.dy = lw[k].dy;
      f.dh_final = fin_dh[k]; f.dc_final = fin_dc[k]; f.dh0 = nullptr; f.dc0 = nullptr;
      f.dX = (k == 2) ? dtop : lw[k - 1].dy; f.dx_beta = 0; f.dx_keep = drop ? keep_enc[k] : nullptr; f.dUb = dub;
      return f;
    };
    // layer 1: top = y_f + y_b so both directions receive dtop (layers.py:176-180)
    auto l1_scan = [&](bool bwd_dir, void* dub) {
      BwdScan f;
      f.l = bwd_dir ? 1 : 0; f.X = Xs; f.din = E; f.steps = S; f.reverse = bwd_dir; f.mask = src_mask_d; f.dy = dtop;
      f.dh_final = bwd_dir ? fin_dh[1] : nullptr; f.dc_final = bwd_dir ? fin_dc[1] : nullptr;
      f.dh0 = nullptr; f.dc0 = nullptr; f.dX = dXemb; f.dx_beta = bwd_dir ? 0 : 1; f.dx_keep = nullptr; f.dUb = dub;
      return f;
    };
    auto single = [&](const BwdScan& f) {
      if (single_bwd_rows()) { bwd_single(f); return; }
      scan_bwd(f.l, f.X, f.din, f.steps, f.reverse, f.mask, f.dy, f.dh_final, f.dc_final, f.dh0, f.dc0, f.dX,
               f.dx_beta, f.dx_keep);
    };
    if (use_dual_bwd()) {
      // pairs of independent scans: dL alone, then (d(k), e(k+1)) for k = L-1..1, then (e1 bwd, e1 fwd);
      // with the dW split, each level's scans write their own dU (the deferred
      // columns are read while the next level runs) and every level but the
      // last leaves its first bg_cols() dW columns to the background stream
      const int nb = bg_cols();
      auto dub = [&](int l, void* fb) { return nb ? dUl[l] : fb; };
      BwdScan dl = dec_scan(L, dub(2 * L, dU));
      bwd_single(dl, false);
      bwd_post(dl, nb);
      bwd_dw_bg(dl);
      for (int k = L - 1; k >= 1; --k) {
        BwdScan d = dec_scan(k, dub(L + k, dU)), e = enc_scan(k + 1, dub(k + 1, dU2));
        bwd_pair(d, e);
        if (use_overlap()) {  // disjoint outputs: the encoder scan's GEMMs on the side stream
          fork();
          bwd_post(d, nb);
          on_side_stream([&]() { bwd_post(e, nb); });
          join();
        } else {
          bwd_post(d, nb);
          bwd_post(e, nb);
        }
        bwd_dw_bg(d);
        bwd_dw_bg(e);
      }
      // the target table's rows are final once dec.l1's input grads are: in
      // data parallel their exchange overlaps the enc.l1 scans
      if (dp && n_tables == 2) embed_grads(1, dp);
      BwdScan b1 = l1_scan(true, dub(1, dU)), f1 = l1_scan(false, dub(0, dU2));
      bwd_pair(b1, f1);
      if (use_overlap()) {
        // weight grads of both directions overlap; the two dX GEMMs stay ordered
        // (enc.l1.fwd accumulates into enc.l1.bwd's embedding grads)
        fork();
        bwd_post(b1);
        BwdScan f1w = f1;
        f1w.dX = nullptr;
        on_side_stream([&]() { bwd_post(f1w); });
        join();
        bwd_post_dx(f1);
      } else {
        bwd_post(b1);
        bwd_post(f1);
      }
    } else {
      for (int k = L; k >= 1; --k) single(dec_scan(k, dU));
      for (int k = L; k >= 2; --k) single(enc_scan(k, dU));
      single(l1_scan(true, dU));
      single(l1_scan(false, dU));
    }
    for (int t = 0; t < n_tables; ++t) embed_grads(t, dp);
    bg_join();  // the deferred weight-gradient columns, before the norm

    // ===== data parallel: sum grads / loss / status over ranks (NCCL) =====
    if (dp) {
      if (ar_buckets) {
        for (int id = 0; id < (int)layers.size() + 2; ++id) allreduce_region(id);  // any not yet issued
      } else {
        allreduce(dg, dense_n, NCCL_FLOAT32);
      }
      allreduce(losssum_d, 1, NCCL_FLOAT64);
      // the status word is a set of flags: spread it one flag per int, take the
      // max over ranks and rebuild it (a SUM of the words carries between flags)
      status_spread_kernel<<<1, 32, 0, st>>>(status_d, out_d->flag4);
      CMT_LAUNCHED(); tl_mark(st, "status_spread_kernel");
      allreduce(out_d->flag4, ST_NFLAGS, NCCL_INT32, NCCL_MAX);
      allreduce_join();
      status_gather_kernel<<<1, 32, 0, st>>>(out_d->flag4, status_d);
      CMT_LAUNCHED(); tl_mark(st, "status_gather_kernel");
    }
    // ===== global-norm clip + SGD (training.py:123-142) =====
    int nparts = 0;
    for (const GradSeg& sg : segs) {
      sumsq_partial_kernel<<<NORM_BLOCKS, 256, 0, st>>>(dg + sg.off, (long long)sg.n, normpart + nparts, sg.lanes);
      CMT_LAUNCHED(); tl_mark(st, "sumsq_partial_kernel");
      nparts += NORM_BLOCKS;
    }
    for (int t = 0; t < n_tables; ++t) {
      const int rows = dp ? nunion[t] : rows_grid(t);
      if (!table_learn[t] || rows == 0) continue;
      const float* gsrc = dp ? ubuf[t] : gcomp[t];
      long long gn = (long long)rows * E;
      sumsq_partial_kernel<<<NORM_BLOCKS, 256, 0, st>>>(gsrc, gn, normpart + nparts, 15, dp ? nullptr : rows_dev(t), E);
      CMT_LAUNCHED(); tl_mark(st, "sumsq_partial_kernel");
      nparts += NORM_BLOCKS;
    }
    clip_scale_kernel<<<1, CLIP_THREADS, 0, st>>>(normpart, nparts, scal_d, normscal_d, s32_d, status_d);
    CMT_LAUNCHED(); tl_mark(st, "clip_scale_kernel");
    if (!(a.flags & CMT_FLAG_NO_UPDATE)) {
      for (const GradSeg& sg : segs) {
        ncu_begin(10);
        sgd_dense_kernel<<<grid_for((long long)sg.n), 256, 0, st>>>(dw + sg.off, dg + sg.off,
                                                                    bf ? dsh + sg.off : nullptr, (long long)sg.n,
                                                                    s32_d, status_d, sg.lanes);
        ncu_end();
        CMT_LAUNCHED(); tl_mark(st, "sgd_dense_kernel");
      }
      for (int t = 0; t < n_tables; ++t) {
        if (!table_learn[t]) continue;
        if (dp) {  // the union rows, identical on every rank
          if (nunion[t] == 0) continue;
          sgd_rows_kernel<<<nunion[t], 128, 0, st>>>(emb_w[t], bf ? emb_sh[t] : nullptr, E, uids_d[t], nunion[t],
                                                      ubuf[t], s32_d, status_d);
          CMT_LAUNCHED(); tl_mark(st, "sgd_rows_kernel");
          continue;
        }
        if (rows_grid(t) == 0) continue;
        sgd_rows_kernel<<<rows_grid(t), 128, 0, st>>>(emb_w[t], bf ? emb_sh[t] : nullptr, E, uniq_d[t], nuniq[t],
                                                       gcomp[t], s32_d, status_d, rows_dev(t));
        CMT_LAUNCHED(); tl_mark(st, "sgd_rows_kernel");
      }
    }
    CMT_CUDA(cudaGetLastError());
    CMT_CUDA(cudaMemcpyAsync(out_h, out_d, sizeof(StepOut), cudaMemcpyDeviceToHost, st));
    return draw;
  }
  // debug: copy an internal buffer (converted to fp32) to the host
  long long debug_buffer(const std::string& name, float* out, long long cap) {
    CMT_CUDA(cudaStreamSynchronize(st));
    long long NS = (long long)S * B, NT = (long long)T * B;
    const void* p = nullptr;
    long long n = 0;
    bool act = false;
    auto lidx = [&](const std::string& s) { return std::stoi(s.substr(s.find(':') + 1)); };
    if (name == "Xs") { p = Xs; n = NS * E; act = true; }
    else if (name == "Xt") { p = Xt; n = NT * E; act = true; }
    else if (name == "top") { p = top; n = NS * H; act = true; }
    else if (name == "u_att") { p = u_att; n = NT * H; act = true; }
    else if (name == "cst_att") { p = cst_att; n = NT * 2 * H; act = true; }
    else if (name == "hod") { p = hod; n = NT * H; act = true; }
    else if (name == "Y") { p = Y; n = NT * V; act = true; }
    else if (name == "dhpre") { p = dhpre; n = NT * H; act = true; }
    else if (name == "du_att") { p = du_att; n = NT * H; act = true; }
    else if (name == "alpha") { p = alpha; n = (long long)B * T * S; }
    else if (name == "ho") { p = ho; n = NT * H; }
    else if (name == "dcst") { p = dcst; n = NT * 2 * H; }
    else if (name == "dXemb") { p = dXemb; n = (NS + NT) * E; }
    else if (name == "dtop") { p = dtop; n = NS * H; }
    else if (name.rfind("yext:", 0) == 0) { int l = lidx(name); p = lw[l].yext; n = ((l <= L ? S : T) + 1LL) * B * H; act = true; }
    else if (name.rfind("cext:", 0) == 0) { int l = lidx(name); p = lw[l].cext; n = ((l <= L ? S : T) + 1LL) * B * H; }
    else if (name.rfind("acts:", 0) == 0) { int l = lidx(name); p = lw[l].acts; n = (l <= L ? S : T) * (long long)B * 4 * H; }
    else if (name.rfind("dy:", 0) == 0) { int l = lidx(name); p = lw[l].dy; n = (l <= L ? S : T) * (long long)B * H; }
    else throw Error(CMT_ERR_CONFIG, "unknown debug buffer " + name);
    if (n > cap) throw Error(CMT_ERR_SHAPE, "debug buffer too small");
    if (act && bf) {
      std::vector<bf16> tmp(n);
      copy_sync(tmp.data(), p, n * 2, cudaMemcpyDeviceToHost);
      for (long long i = 0; i < n; ++i) out[i] = __bfloat162float(tmp[i]);
    } else {
      copy_sync(out, p, n * 4, cudaMemcpyDeviceToHost);
    }
    return n;
  }
  unsigned long long last_draws = 0;
  double last_ntok = 1;
  int time_dominant = 0;  // bit c: CUDA-event probes around the launches of kernel class c
  int stop_after = 0;  // debug: 1 = after the logits GEMM, 2 = after the CE
  // probes (bench.py's roofline, timed inside the timed steps on the launching
  // stream): class 0 the logits GEMM, 1 the BPTT scan launches, 2 the forward scan launches
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> probe_ev[3];
  // ncu_class >= 0: the first launch of that class runs inside
  // cudaProfilerStart/Stop, so `ncu --profile-from-start off -c 1` captures it
  // (scripts/ncu_step.py): 0 logits GEMM, 1 BPTT scan, 2 forward scan, 3 Ux GEMM,
  // 4 dX GEMM, 5 dW GEMM, 6 ce_stats, 7 ce_grad, 8 dropout, 9 attention scores
  // GEMM, 10 dense SGD, 11 dW_o GEMM, 12 embedding scatter
  int ncu_class = -1, ncu_skip = 0;  // ncu_skip: launches of the class to pass over first
  bool ncu_on = false, ncu_done = false;
  void ncu_begin(int cls) {
    if (cls != ncu_class || ncu_done) return;
    if (ncu_skip > 0) {
      --ncu_skip;
      return;
    }
    CMT_CUDA(cudaProfilerStart());
    ncu_on = true;
  }
  void ncu_end() {
    if (!ncu_on) return;
    CMT_CUDA(cudaProfilerStop());
    ncu_on = false;
    ncu_done = true;
  }
  std::vector<cudaEvent_t> ev_pool;  // probe events, reused (destroyed with the engine)
  cudaEvent_t pooled_event() {
    if (ev_pool.empty()) {
      cudaEvent_t e;
      CMT_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
  cudaEvent_t probe_begin(int cls) {
    ncu_begin(cls);
    if (!((time_dominant >> cls) & 1)) return nullptr;
    cudaEvent_t e0 = capturing ? nullptr : pooled_event();
    if (capturing) CMT_CUDA(cudaEventCreate(&e0));  // owned by the captured graph
    // inside a capture the record becomes a graph node (its event is swapped per replay)
    CMT_CUDA(cudaEventRecordWithFlags(e0, st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
    return e0;
  }
  void probe_end(int cls, cudaEvent_t e0) {
    ncu_end();
    if (!e0) return;
    cudaEvent_t e1 = capturing ? nullptr : pooled_event();
    if (capturing) CMT_CUDA(cudaEventCreate(&e1));
    CMT_CUDA(cudaEventRecordWithFlags(e1, st, capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
    if (capturing) cap_probes.push_back({cls, {e0, e1}});
    else probe_ev[cls].push_back({e0, e1});
  }
  // mean duration (ms) of the probed launches of class cls since the last call
  double probe_ms(int cls, double* count) {
    if (cls < 0 || cls > 2) throw Error(CMT_ERR_CONFIG, "probe class out of range");
    CMT_CUDA(cudaStreamSynchronize(st));
    double tot = 0;
    for (auto& p : probe_ev[cls]) {
      float ms = 0;
      CMT_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
      tot += ms;
      // back to the pool, not destroyed: a replayed graph's record nodes may
      // still name them until their next replay swaps in other events
      ev_pool.push_back(p.first);
      ev_pool.push_back(p.second);
    }
    *count = (double)probe_ev[cls].size();
    double r = probe_ev[cls].empty() ? 0.0 : tot / probe_ev[cls].size();
    probe_ev[cls].clear();
    return r;
  }

  void wait(cmt_step_result* res) {
    CMT_CUDA(cudaStreamSynchronize(st));
    res->draws = last_draws;
    res->loss = (double)((float)out_h->loss_sum / (float)last_ntok);
    res->loss_sum = out_h->loss_sum;
    res->ntok = last_ntok;
    res->grad_norm = out_h->scal[1];
    int s = out_h->status;
    if (last_infer) s &= ~ST_LOSS;  // dev_entropy does not check the loss (training.py:174-181)
    res->status = (s & ST_HANG)   ? CMT_ERR_INTERNAL
                : (s & ST_SCORES) ? CMT_ERR_NUM_SCORES
                : (s & ST_LOGITS) ? CMT_ERR_NUM_LOGITS
                : (s & ST_LOSS)   ? CMT_ERR_NUM_LOSS
                : (s & ST_NORM)   ? CMT_ERR_NUM_NORM
                                  : CMT_OK;
  }
};

}  // namespace cmt

// ===========================================================================
// C ABI
// ===========================================================================
using cmt::Engine;
using cmt::Error;

struct cmt_engine {
  Engine* eng;
  std::string err;
};
static thread_local std::string g_err;

template <class F>
static int guard(cmt_engine* e, F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& x) {
    (e ? e->err : g_err) = x.what();
    return x.code;
  } catch (const std::exception& x) {
    (e ? e->err : g_err) = x.what();
    return cmt::CMT_ERR_INTERNAL;
  }
}

extern "C" {

int cmt_create(const cmt_config* cfg, int device, cmt_engine** out) {
  return guard(nullptr, [&] {
    auto* h = new cmt_engine;
    try {
      h->eng = new Engine(*cfg, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void cmt_destroy(cmt_engine* e) {
  if (!e) return;
  delete e->eng;
  delete e;
}
const char* cmt_last_error(cmt_engine* e) { return e ? e->err.c_str() : g_err.c_str(); }
int cmt_num_blocks(cmt_engine* e) { return (int)e->eng->blocks.size(); }
int cmt_block_info(cmt_engine* e, int idx, char* name, int cap, long long* rows, long long* cols) {
  return guard(e, [&] {
    if (idx < 0 || idx >= (int)e->eng->blocks.size()) throw Error(cmt::CMT_ERR_SHAPE, "block index out of range");
    auto& b = e->eng->blocks[idx];
    std::snprintf(name, cap, "%s", b.name.c_str());
    *rows = b.rows;
    *cols = b.cols;
  });
}
int cmt_upload_param(cmt_engine* e, int idx, const float* h, long long rows, long long cols) {
  return guard(e, [&] { e->eng->upload(idx, h, rows, cols); });
}
int cmt_download_param(cmt_engine* e, int idx, float* h, long long rows, long long cols) {
  return guard(e, [&] { e->eng->download(idx, h, rows, cols, false); });
}
int cmt_snapshot_save(cmt_engine* e, int slot) {
  return guard(e, [&] { e->eng->snapshot_save(slot); });
}
int cmt_snapshot_restore(cmt_engine* e, int slot) {
  return guard(e, [&] { e->eng->snapshot_restore(slot); });
}
int cmt_snapshot_free(cmt_engine* e, int slot) {
  return guard(e, [&] { e->eng->snapshot_free(slot); });
}
int cmt_snapshot_download(cmt_engine* e, int slot, int idx, float* h, long long rows, long long cols) {
  return guard(e, [&] {
    e->eng->check_slot(slot);
    e->eng->download(idx, h, rows, cols, false, slot);
  });
}
int cmt_beam_begin(cmt_engine* e, const long long* src_ids, const float* src_mask, int S, int B, int beam,
                   int n_best, const int* max_len, const double* lp_table, int lp_table_len) {
  return guard(e, [&] { e->eng->beam_begin(src_ids, src_mask, S, B, beam, n_best, max_len, lp_table, lp_table_len); });
}
int cmt_beam_step(cmt_engine* e, int max_steps, int* n_active) {
  return guard(e, [&] { *n_active = e->eng->beam_step(max_steps); });
}
int cmt_beam_result(cmt_engine* e, int b, int rank, int* tokens, int cap, int* n_tokens, double* score,
                    double* log_prob, int* truncated, int* n_results) {
  return guard(e, [&] { *n_results = e->eng->beam_result(b, rank, tokens, cap, n_tokens, score, log_prob, truncated); });
}
int cmt_set_learnable(cmt_engine* e, int idx, int learnable) {
  return guard(e, [&]() { e->eng->set_learnable(idx, learnable != 0); });
}
int cmt_status_combine(const int* words, int n) { return cmt::status_combine(words, n); }
int cmt_staged_rows(cmt_engine* e, int table, int* ids, int cap, int* n) {
  return guard(e, [&] {
    cmt::Engine& g = *e->eng;
    if (table < 0 || table >= g.n_tables) throw Error(cmt::CMT_ERR_SHAPE, "table index out of range");
    g.host_segments(table);
    *n = (int)g.uniq_h[table].size();
    if (ids) {
      if (cap < *n) throw Error(cmt::CMT_ERR_SHAPE, "id buffer too small");
      std::memcpy(ids, g.uniq_h[table].data(), g.uniq_h[table].size() * 4);
    }
  });
}
int cmt_set_union(cmt_engine* e, int table, const int* ids, int n) {
  return guard(e, [&] { e->eng->set_union(table, ids, n); });
}
int cmt_download_grad(cmt_engine* e, int idx, float* h, long long rows, long long cols) {
  return guard(e, [&] { e->eng->download(idx, h, rows, cols, true); });
}
int cmt_stage_batch(cmt_engine* e, const long long* src, const float* sm, int S, const long long* tgt, const float* tm,
                    int T, int B) {
  return guard(e, [&] { e->eng->stage(src, sm, S, tgt, tm, T, B); });
}
int cmt_run_step(cmt_engine* e, const cmt_step_args* a, cmt_step_result* r) {
  int rc = guard(e, [&] { e->eng->run(*a, r); });
  if (rc == 0 && r && !(a->flags & CMT_FLAG_ASYNC) && r->status != 0) {
    e->err = r->status == CMT_ERR_INTERNAL ? "recurrent scan flag wait timed out (step aborted, weights unchanged)"
                                           : "numeric error in train step";
    return r->status;
  }
  return rc;
}
int cmt_train_step(cmt_engine* e, const long long* src, const float* sm, int S, const long long* tgt, const float* tm,
                   int T, int B, const cmt_step_args* a, cmt_step_result* r) {
  int rc = cmt_stage_batch(e, src, sm, S, tgt, tm, T, B);
  if (rc) return rc;
  return cmt_run_step(e, a, r);
}
int cmt_wait(cmt_engine* e, cmt_step_result* r) {
  int rc = guard(e, [&] { e->eng->wait(r); });
  if (!rc && r->status == CMT_ERR_INTERNAL) e->err = "recurrent scan flag wait timed out (step aborted, weights unchanged)";
  return rc ? rc : r->status;
}
int cmt_set_comm(cmt_engine* e, const void* uid, int rank, int world) {
  return guard(e, [&] { e->eng->set_comm(uid, rank, world); });
}
int cmt_nccl_unique_id(void* out128) {
  return guard(nullptr, [&] {
    cmt::g_nccl.load();
    int r = cmt::g_nccl.get_unique_id(out128);
    if (r) throw Error(cmt::CMT_ERR_CUDA, "ncclGetUniqueId failed");
  });
}
int cmt_event_record(cmt_engine* e, int slot) {
  return guard(e, [&] { CMT_CUDA(cudaEventRecord(e->eng->ev[slot & 15], e->eng->st)); });
}
int cmt_event_elapsed(cmt_engine* e, int a, int b, float* ms) {
  return guard(e, [&] {
    CMT_CUDA(cudaEventSynchronize(e->eng->ev[b & 15]));
    CMT_CUDA(cudaEventElapsedTime(ms, e->eng->ev[a & 15], e->eng->ev[b & 15]));
  });
}
unsigned long long cmt_launch_count(void) { return cmt::g_launches; }

// ---- test hooks (not part of the reference interface): single kernels on device pointers ----
int cmt_test_gemm(int mode, int M, int N, int K, const void* A, long long lda, int a_mn, const void* B, long long ldb,
                  int b_mn, void* C, long long ldc, int bn, int flags, const float* bias) {
  return guard(nullptr, [&] {
    cmt::EpiStore e;
    e.C = C; e.ldc = ldc; e.beta = flags & 1; e.c_bf16 = (flags >> 1) & 1; e.act = (flags >> 2) & 1; e.bias = bias;
    cmt::Mat a{A, lda, a_mn}, b{B, ldb, b_mn};
    cudaStream_t st = 0;
    if (mode == CMT_MODE_BF16 && K < cmt::tc::BK) {  // same routing as the engine
      dim3 grid(cmt::ceil_div(N, 64), cmt::ceil_div(M, 64));
      cmt::gemm_simt_kernel<cmt::EpiStore, cmt::bf16><<<grid, 256, 0, st>>>((const cmt::bf16*)A, lda, a_mn,
                                                                             (const cmt::bf16*)B, ldb, b_mn, M, N, K, e);
    } else if (mode == CMT_MODE_FP32) {
      dim3 grid(cmt::ceil_div(N, 64), cmt::ceil_div(M, 64));
      cmt::gemm_simt_kernel<cmt::EpiStore><<<grid, 256, 0, st>>>((const float*)A, lda, a_mn, (const float*)B, ldb, b_mn,
                                                                   M, N, K, e);
    } else {
      int key = a_mn * 2 + b_mn;
#define T_(BN_, AMN, BMN, CG_) else if (bn == BN_ + CG_ - 1 && key == AMN * 2 + BMN) cmt::launch_tc<BN_, AMN, BMN, cmt::EpiStore, CG_>(st, M, N, K, a, b, e);
      if (0) {}
      T_(64, 0, 1, 1) T_(128, 0, 1, 1) T_(256, 0, 1, 1) T_(64, 0, 0, 1) T_(128, 0, 0, 1) T_(256, 0, 0, 1) T_(64, 1, 1, 1)
      T_(128, 1, 1, 1) T_(256, 1, 1, 1)
      T_(128, 0, 1, 2) T_(256, 0, 1, 2) T_(128, 0, 0, 2) T_(256, 0, 0, 2) T_(128, 1, 1, 2) T_(256, 1, 1, 2)
      else throw Error(cmt::CMT_ERR_INTERNAL, "no such GEMM instantiation");
#undef T_
    }
    CMT_CUDA(cudaGetLastError());
    CMT_CUDA(cudaDeviceSynchronize());
  });
}
int cmt_test_dropout(unsigned long long sh, unsigned long long sl, unsigned long long ih, unsigned long long il,
                     unsigned long long base, int N, int H, double p, const float* x, float* y, unsigned char* keep) {
  return guard(nullptr, [&] {
    cmt::Pcg pcg{sh, sl, ih, il};
    dim3 blk(32, 8), grid(cmt::ceil_div(H, 32), cmt::ceil_div(cmt::ceil_div(N, 32), 8));
    (void)grid;
    cmt::PcgJump* jt = nullptr;
    CMT_CUDA(cudaMalloc(&jt, sizeof(cmt::PcgJump) + sizeof(cmt::Pcg)));
    cmt::Pcg* pcg_d = (cmt::Pcg*)(jt + 1);
    CMT_CUDA(cudaMemcpy(pcg_d, &pcg, sizeof(pcg), cudaMemcpyHostToDevice));
    cmt::pcg_jump_table_kernel<<<1, 1>>>(jt, ih, il);
    dim3 grid4(cmt::ceil_div(H, 32), cmt::ceil_div(cmt::ceil_div(N, cmt::DROP4_DPT), 8));
    cmt::dropout_fwd_kernel4<float, float><<<grid4, blk>>>(x, y, keep, N, H, pcg_d, jt, base, cmt::dropout_threshold(p),
                                                            1.0f / (float)(1.0 - p));
    cudaError_t err = cudaDeviceSynchronize();
    cudaFree(jt);
    CMT_CUDA(err);
    CMT_CUDA(cudaGetLastError());
    CMT_CUDA(cudaDeviceSynchronize());
  });
}
int cmt_set_option(cmt_engine* e, const char* key, long long value) {
  return guard(e, [&] {
    std::string k(key);
    if (k == "time_dominant") e->eng->time_dominant = (int)value;
    else if (k == "ncu_skip") e->eng->ncu_skip = (int)value;
    else if (k == "bwd_bg") {
      if (e->eng->staged) throw Error(cmt::CMT_ERR_CONFIG, "set bwd_bg before staging a batch");
      e->eng->bwd_bg = (int)value;
    }
    else if (k == "ncu_class") {
      e->eng->ncu_class = (int)value;
      e->eng->ncu_done = false;
    } else if (k == "att_tc") {
      if (e->eng->staged) throw Error(cmt::CMT_ERR_CONFIG, "set att_tc before staging a batch");
      e->eng->att_tc = (int)value;
    }
    else if (k == "persistent") e->eng->persistent = (int)value;
    else if (k == "cg2") e->eng->cg2 = (int)value;
    else if (k == "dual") e->eng->dual = (int)value;
    else if (k == "fwd_tm") e->eng->fwd_tm = (int)value;
    else if (k == "ar_overlap") e->eng->ar_overlap = (int)value;
    else if (k == "early_dec1") e->eng->early_dec1 = (int)value;
    else if (k == "att_split") e->eng->att_split = (int)value;
    else if (k == "allow_empty_targets") e->eng->allow_empty_targets = (int)value;
    else if (k == "overlap") e->eng->overlap = (int)value;
    else if (k == "ce2") {
      if (e->eng->staged && (value != 0) != (e->eng->ce2 != 0)) throw Error(cmt::CMT_ERR_CONFIG, "set ce2 before staging");
      e->eng->ce2 = (int)value;
    }
    else if (k == "tma_store") cmt::g_tma_store = (int)value;
    else if (k == "gemm_opt") cmt::g_gemm_opt = (int)value;
    else if (k == "splitk") cmt::g_splitk = (int)value;
    else if (k == "timeline") {
      cmt::g_tl.on = value != 0;
      for (auto& m : cmt::g_tl.marks) cudaEventDestroy(m.second);
      cmt::g_tl.marks.clear();
    }
    else if (k == "trace_layer") {
      e->eng->trace_layer = (int)value;
      if (!e->eng->trace_d) CMT_CUDA(cudaMalloc(&e->eng->trace_d, 4096 * 8));
      CMT_CUDA(cudaMemset(e->eng->trace_d, 0, 4096 * 8));
    }
    else if (k == "stop_after") e->eng->stop_after = (int)value;
    else if (k == "graph") e->eng->use_graph = (int)value;
    else if (k == "seg_dev") e->eng->use_seg_dev = (int)value;
    else if (k == "mask_ahead") e->eng->mask_ahead = (int)value;
    else throw Error(cmt::CMT_ERR_CONFIG, "unknown option " + k);
    // options select launch configurations: captured steps are re-captured
    if (e && e->eng) {
      CMT_CUDA(cudaStreamSynchronize(e->eng->st));
      e->eng->drop_graphs();
    }
  });
}
// Timeline of the launches recorded since the option "timeline" was set:
// "label<TAB>ms" per launch (ms since the previous mark), newline separated.
int cmt_timeline(cmt_engine* e, char* buf, long long cap) {
  return guard(e, [&] {
    CMT_CUDA(cudaDeviceSynchronize());
    std::string out;
    auto& mk = cmt::g_tl.marks;
    for (size_t i = 1; i < mk.size(); ++i) {
      if (mk[i].first == "<start>") continue;
      float ms = 0;
      CMT_CUDA(cudaEventElapsedTime(&ms, mk[i - 1].second, mk[i].second));
      out += mk[i].first + "\t" + std::to_string(ms) + "\n";
    }
    for (auto& m : mk) cudaEventDestroy(m.second);
    mk.clear();
    if ((long long)out.size() + 1 > cap) throw Error(cmt::CMT_ERR_SHAPE, "timeline buffer too small");
    memcpy(buf, out.c_str(), out.size() + 1);
  });
}
int cmt_debug_buffer(cmt_engine* e, const char* name, float* out, long long cap, long long* n) {
  return guard(e, [&] { *n = e->eng->debug_buffer(name, out, cap); });
}
int cmt_get_stat(cmt_engine* e, const char* key, double* value, double* count) {
  return guard(e, [&] {
    std::string k(key);
    if (k == "dominant_ms") *value = e->eng->probe_ms(0, count);
    else if (k.rfind("stage_us:", 0) == 0) {
      int i = std::stoi(k.substr(9)) & 7;
      *value = e->eng->stage_us[i];
      *count = e->eng->stage_us[7];
      e->eng->stage_us[i] = 0;
    }
    else if (k == "graph_replays") { *value = (double)e->eng->graph_replays; *count = (double)e->eng->graphs.size(); }
    else if (k.rfind("probe_ms:", 0) == 0) *value = e->eng->probe_ms(std::stoi(k.substr(9)), count);
    else if (k.rfind("trace:", 0) == 0) {
      int i = std::stoi(k.substr(6));
      unsigned long long v = 0;
      CMT_CUDA(cudaStreamSynchronize(e->eng->st));
      CMT_CUDA(cudaMemcpy(&v, e->eng->trace_d + i, 8, cudaMemcpyDeviceToHost));
      *value = (double)v;
    }
    else throw Error(cmt::CMT_ERR_CONFIG, "unknown stat " + k);
  });
}

}  // extern "C"
