/*
 * cytonmt_b200.h — C ABI of the B200-native CytonMT train-step engine.
 *
 * The reference has no FFI: its only operator interface is the Python
 * train step `minmt.training.train_step(model, batch, cfg, lr, rng) -> float`
 * (/root/reference/pkg/src/minmt/training.py:145-159) built on the Layer
 * contract (graph.py:34-62).  These entry points are what a ctypes (or cgo /
 * JNI) binding of that function needs; the Python drop-in in
 * paper_1802_07170_b200/training.py binds them.
 *
 * All pointers are plain host pointers; no torch types cross the boundary.
 * Every function returns 0 on success or a cmt_status code; the message of the
 * last failure is available from cmt_last_error().
 */
#ifndef CYTONMT_B200_H
#define CYTONMT_B200_H
#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* status codes (mapped to the reference's exception types by the wrapper) */
enum cmt_status {
  CMT_OK = 0,
  CMT_ERR_CONFIG = 1,      /* ConfigError: bad token id (model.py:146-151), empty target mask (training.py:108-110) */
  CMT_ERR_MASK = 2,        /* MaskError: fully masked source column (attention.py:153-154) */
  CMT_ERR_SHAPE = 3,       /* ShapeError */
  CMT_ERR_NUM_SCORES = 4,  /* NumericError: non-finite attention scores (tensor.py:139-140) */
  CMT_ERR_NUM_LOGITS = 5,  /* NumericError: non-finite logits (tensor.py:148-149) */
  CMT_ERR_NUM_LOSS = 6,    /* NumericError: non-finite loss (training.py:154-155) */
  CMT_ERR_NUM_NORM = 7,    /* NumericError: non-finite grad norm (training.py:133-134) */
  CMT_ERR_CUDA = 8,
  CMT_ERR_INTERNAL = 9
};

/* precision modes */
enum cmt_mode {
  CMT_MODE_FP32 = 0, /* fp32 validation mode: fp32 SIMT GEMMs, 1e-4 parity */
  CMT_MODE_BF16 = 1  /* production: tcgen05 bf16 GEMMs, fp32 accumulate/state, 2e-2 parity */
};

/* step flags */
enum cmt_flags {
  CMT_FLAG_NO_UPDATE = 1, /* compute loss + grads, skip clip/SGD (grads kept for cmt_download_grad) */
  CMT_FLAG_ASYNC = 2,     /* do not wait for the step; result filled by cmt_wait() */
  CMT_FLAG_INFER = 4      /* forward only in INFER mode (no dropout, no backward, no update):
                             the dev_entropy pass of training.py:162-182 (use epsilon = 0) */
};

/* mirrors ModelConfig (model.py:46-62) */
typedef struct {
  int vocab_size, embedding_size, hidden_size, depth;
  int output_tanh, shared_embeddings;
  double dropout;
  int mode; /* cmt_mode */
} cmt_config;

/* per-step arguments: TrainConfig fields used by train_step + the dropout RNG */
typedef struct {
  double lr;          /* learning rate (train_step arg) */
  double clip_norm;   /* TrainConfig.grad_clip_norm; < 0 (or NaN) means None; 0 clips to a zero step */
  double epsilon;     /* TrainConfig.label_smoothing */
  unsigned long long pcg_state_hi, pcg_state_lo, pcg_inc_hi, pcg_inc_lo; /* numpy PCG64 state */
  double global_ntok; /* data-parallel: sum of tgt_mask over all ranks (<= 0: this batch) */
  int flags;          /* cmt_flags */
} cmt_step_args;

typedef struct {
  double loss;                  /* smoothed loss (training.py:113) */
  double grad_norm;             /* global L2 norm before clipping (training.py:128-131) */
  unsigned long long draws;     /* PCG64 doubles consumed by dropout; caller advances its generator */
  int status;                   /* cmt_status of the step */
  double loss_sum;              /* sum over tokens of per-token loss * mask */
  double ntok;                  /* token count the loss is averaged over */
} cmt_step_result;

typedef struct cmt_engine cmt_engine;

int cmt_create(const cmt_config* cfg, int device, cmt_engine** out);
void cmt_destroy(cmt_engine* e);
const char* cmt_last_error(cmt_engine* e);           /* e may be NULL (create failures) */

/* parameter registry in the reference's order (model.py:86-95) */
int cmt_num_blocks(cmt_engine* e);
int cmt_block_info(cmt_engine* e, int idx, char* name, int name_cap, long long* rows, long long* cols);
int cmt_upload_param(cmt_engine* e, int idx, const float* host_rowmajor, long long rows, long long cols);
int cmt_download_param(cmt_engine* e, int idx, float* host_rowmajor, long long rows, long long cols);
int cmt_download_grad(cmt_engine* e, int idx, float* host_rowmajor, long long rows, long long cols);
/* ParamBlock.learnable (graph.py:20-31): a frozen block (learnable = 0) is left
 * out of the global grad norm and the update (training.py:128-139); its grad is
 * still computed (cmt_download_grad).  Every block starts learnable. */
int cmt_set_learnable(cmt_engine* e, int idx, int learnable);

/* GPU translation: batched beam search on the device.
 * The reference translates sentence by sentence, one decode_step per live
 * hypothesis (decoding.py:89-153, model.py:180-236).  cmt_beam_begin encodes a
 * padded batch of B source sentences (ids int64 (S, B) C order, mask float32
 * {0,1}) with the INFER-mode forward and starts one beam of `beam` (<= 32)
 * slots per sentence; max_len[b] = DecodeConfig.cap_for(len) (>= 1);
 * lp_table[n] = length_penalty(n) = ((5 + n) / 6) ** alpha for n in
 * [0, lp_table_len), lp_table_len >= max(max_len) + 2 (computed by the caller
 * so scores are bit-identical to the reference's).  cmt_beam_step runs up to
 * max_steps decoder steps for every unfinished sentence (all live hypotheses of
 * all sentences as the rows of one step) and returns the number of sentences
 * still searching.  Once that is 0, cmt_beam_result returns sentence b's
 * result `rank`: the finished hypotheses ordered by (score desc, arrival
 * asc), at most max(n_best, 1), tokens without the final EOS (*n_results = how
 * many); when nothing finished within max_len, one truncated entry (the best
 * live hypothesis, *truncated = 1, *score = NaN: the caller divides log_prob by
 * length_penalty(max(len, 1)) as decoding.py:150-153).  Greedy decoding is the
 * beam of 1 with alpha = 0 (decoding.py:156-171). */
int cmt_beam_begin(cmt_engine* e, const long long* src_ids, const float* src_mask, int S, int B, int beam,
                   int n_best, const int* max_len, const double* lp_table, int lp_table_len);
int cmt_beam_step(cmt_engine* e, int max_steps, int* n_active);
int cmt_beam_result(cmt_engine* e, int b, int rank, int* tokens, int cap, int* n_tokens, double* score,
                    double* log_prob, int* truncated, int* n_results);

/* device-resident parameter snapshots: replaces the host round trip of
 * ModelParams.copy_data / load_data (model.py:104-115) that the Trainer uses
 * to keep and restore its best parameters (training.py:205, 246-254, 269).
 * slot in [0, 4); save/restore copy the fp32 masters device-to-device (restore
 * also refreshes the bf16 shadows); download reads one block of a saved slot in
 * the reference layout (like cmt_download_param); free releases the slot. */
int cmt_snapshot_save(cmt_engine* e, int slot);
int cmt_snapshot_restore(cmt_engine* e, int slot);
int cmt_snapshot_download(cmt_engine* e, int slot, int idx, float* host_rowmajor, long long rows, long long cols);
int cmt_snapshot_free(cmt_engine* e, int slot);

/* batch (data.py:108-122): ids int64 (steps, batch) C order; masks float32 {0,1} */
int cmt_stage_batch(cmt_engine* e, const long long* src_ids, const float* src_mask, int S,
                    const long long* tgt_ids, const float* tgt_mask, int T, int B);
/* run one train step on the staged batch (inputs already in HBM) */
int cmt_run_step(cmt_engine* e, const cmt_step_args* args, cmt_step_result* res);
/* stage + run: the reference-facing call (host buffers, H2D/D2H inside) */
int cmt_train_step(cmt_engine* e, const long long* src_ids, const float* src_mask, int S,
                   const long long* tgt_ids, const float* tgt_mask, int T, int B,
                   const cmt_step_args* args, cmt_step_result* res);
int cmt_wait(cmt_engine* e, cmt_step_result* res);

/* data parallel: NCCL communicator from a 128-byte ncclUniqueId (from cmt_nccl_unique_id on rank 0).
   Grads, loss and status are summed over ranks inside every step; pass global_ntok in cmt_step_args. */
int cmt_set_comm(cmt_engine* e, const void* nccl_unique_id, int rank, int world);
/* data parallel, embedding rows: the ids (ascending) of table `table` (0 src,
 * 1 tgt; one table when embeddings are shared) that the staged batch touches,
 * *n of them (ids may be NULL to query the count); and, before cmt_run_step,
 * the union of every rank's ids (ascending, unique).  The step all-reduces the
 * embedding grads as rows of that union and updates only those rows (the
 * reference's update touches every row, but rows outside the union have zero
 * gradient: w - s*0 = w).  With one rank the union defaults to the rank's ids. */
int cmt_staged_rows(cmt_engine* e, int table, int* ids, int cap, int* n);
int cmt_set_union(cmt_engine* e, int table, const int* ids, int n);
/* the rule that combines the ranks' status words inside a data-parallel step
 * (flag by flag: a flag is raised iff some rank raised it); host-only, no GPU */
int cmt_status_combine(const int* words, int n);
int cmt_nccl_unique_id(void* out128);

/* timing / introspection */
int cmt_event_record(cmt_engine* e, int slot);               /* slot 0..15 on the engine stream */
int cmt_event_elapsed(cmt_engine* e, int a, int b, float* ms);
unsigned long long cmt_launch_count(void);                   /* kernels launched by this library */
int cmt_set_option(cmt_engine* e, const char* key, long long value); /* "time_dominant": CUDA-event the logits GEMM */
int cmt_get_stat(cmt_engine* e, const char* key, double* value, double* count); /* "dominant_ms": mean launch ms */

/* debug: copy an internal buffer (e.g. "Y", "yext:3", "dy:0") as fp32; *n = element count */
/* debug: per-launch device times ("label\tms\n") recorded since set_option("timeline", 1) */
int cmt_timeline(cmt_engine* e, char* buf, long long cap);
int cmt_debug_buffer(cmt_engine* e, const char* name, float* out, long long cap, long long* n);
/* test hooks (parity tests only; device pointers): one GEMM C = A B^T (fp32 out), one dropout site */
/* flags: 1 = accumulate into C, 2 = bf16 C, 4 = tanh; bias may be NULL */
int cmt_test_gemm(int mode, int M, int N, int K, const void* A, long long lda, int a_mn, const void* B, long long ldb,
                  int b_mn, void* C, long long ldc, int bn /* BN; BN+1: CTA-pair tile */, int flags, const float* bias);
int cmt_test_dropout(unsigned long long state_hi, unsigned long long state_lo, unsigned long long inc_hi,
                     unsigned long long inc_lo, unsigned long long base, int N, int H, double p, const float* x,
                     float* y, unsigned char* keep);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif
