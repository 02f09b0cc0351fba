"""ctypes binding of the C ABI in include/cytonmt_b200.h.

The shared library is built in-tree (``paper_1802_07170_b200/libcytonb200.so``)
by ``__graft_entry__.build()`` / ``make -C paper_1802_07170_b200/csrc``.  There
is no fallback: if the library is missing or fails to load, importing the
engine raises.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CMT_LIB: an alternative build of the same library (A/B timing of two builds)
LIB_PATH = os.environ.get("CMT_LIB") or os.path.join(HERE, "libcytonb200.so")

CMT_OK = 0
CMT_ERR_CONFIG = 1
CMT_ERR_MASK = 2
CMT_ERR_SHAPE = 3
CMT_ERR_NUM_SCORES = 4
CMT_ERR_NUM_LOGITS = 5
CMT_ERR_NUM_LOSS = 6
CMT_ERR_NUM_NORM = 7
CMT_ERR_CUDA = 8
CMT_ERR_INTERNAL = 9

MODE_FP32 = 0
MODE_BF16 = 1
FLAG_NO_UPDATE = 1
FLAG_ASYNC = 2
FLAG_INFER = 4

# every symbol include/cytonmt_b200.h declares
EXPORTS = [
    "cmt_create", "cmt_destroy", "cmt_last_error", "cmt_num_blocks", "cmt_block_info",
    "cmt_upload_param", "cmt_download_param", "cmt_download_grad", "cmt_stage_batch",
    "cmt_run_step", "cmt_train_step", "cmt_wait", "cmt_set_comm", "cmt_nccl_unique_id", "cmt_event_record",
    "cmt_event_elapsed", "cmt_launch_count", "cmt_set_option", "cmt_get_stat", "cmt_debug_buffer", "cmt_test_gemm", "cmt_test_dropout", "cmt_timeline",
    "cmt_snapshot_save", "cmt_snapshot_restore", "cmt_snapshot_download", "cmt_snapshot_free",
    "cmt_beam_begin", "cmt_beam_step", "cmt_beam_result", "cmt_set_learnable", "cmt_status_combine",
    "cmt_staged_rows", "cmt_set_union",
]


class Config(ctypes.Structure):
    _fields_ = [("vocab_size", ctypes.c_int), ("embedding_size", ctypes.c_int),
                ("hidden_size", ctypes.c_int), ("depth", ctypes.c_int),
                ("output_tanh", ctypes.c_int), ("shared_embeddings", ctypes.c_int),
                ("dropout", ctypes.c_double), ("mode", ctypes.c_int)]


class StepArgs(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("clip_norm", ctypes.c_double), ("epsilon", ctypes.c_double),
                ("pcg_state_hi", ctypes.c_ulonglong), ("pcg_state_lo", ctypes.c_ulonglong),
                ("pcg_inc_hi", ctypes.c_ulonglong), ("pcg_inc_lo", ctypes.c_ulonglong),
                ("global_ntok", ctypes.c_double), ("flags", ctypes.c_int)]


class StepResult(ctypes.Structure):
    _fields_ = [("loss", ctypes.c_double), ("grad_norm", ctypes.c_double),
                ("draws", ctypes.c_ulonglong), ("status", ctypes.c_int),
                ("loss_sum", ctypes.c_double), ("ntok", ctypes.c_double)]


_lib = None


def load(path=LIB_PATH):
    """Load (once) and prototype the engine library; raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: the CUDA engine is not built (run `python -c 'import __graft_entry__ as g; g.build()'`)")
    lib = ctypes.CDLL(path)
    P, I, LL, D, VP = ctypes.POINTER, ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p
    fp = P(ctypes.c_float)
    llp = P(ctypes.c_longlong)
    lib.cmt_create.argtypes = [P(Config), I, P(VP)]
    lib.cmt_destroy.argtypes = [VP]
    lib.cmt_destroy.restype = None
    lib.cmt_last_error.argtypes = [VP]
    lib.cmt_last_error.restype = ctypes.c_char_p
    lib.cmt_num_blocks.argtypes = [VP]
    lib.cmt_block_info.argtypes = [VP, I, ctypes.c_char_p, I, llp, llp]
    for f in (lib.cmt_upload_param, lib.cmt_download_param, lib.cmt_download_grad):
        f.argtypes = [VP, I, fp, LL, LL]
    for f in (lib.cmt_snapshot_save, lib.cmt_snapshot_restore, lib.cmt_snapshot_free):
        f.argtypes = [VP, I]
    lib.cmt_snapshot_download.argtypes = [VP, I, I, fp, LL, LL]
    dp = P(D)
    lib.cmt_beam_begin.argtypes = [VP, llp, fp, I, I, I, I, P(I), dp, I]
    lib.cmt_beam_step.argtypes = [VP, I, P(I)]
    lib.cmt_beam_result.argtypes = [VP, I, I, P(I), I, P(I), dp, dp, P(I), P(I)]
    lib.cmt_stage_batch.argtypes = [VP, llp, fp, I, llp, fp, I, I]
    lib.cmt_run_step.argtypes = [VP, P(StepArgs), P(StepResult)]
    lib.cmt_train_step.argtypes = [VP, llp, fp, I, llp, fp, I, I, P(StepArgs), P(StepResult)]
    lib.cmt_wait.argtypes = [VP, P(StepResult)]
    lib.cmt_set_comm.argtypes = [VP, VP, I, I]
    lib.cmt_set_learnable.argtypes = [VP, I, I]
    lib.cmt_status_combine.argtypes = [P(I), I]
    lib.cmt_staged_rows.argtypes = [VP, I, P(I), I, P(I)]
    lib.cmt_set_union.argtypes = [VP, I, P(I), I]
    lib.cmt_nccl_unique_id.argtypes = [VP]
    lib.cmt_event_record.argtypes = [VP, I]
    lib.cmt_event_elapsed.argtypes = [VP, I, I, P(ctypes.c_float)]
    lib.cmt_launch_count.argtypes = []
    lib.cmt_launch_count.restype = ctypes.c_ulonglong
    lib.cmt_set_option.argtypes = [VP, ctypes.c_char_p, LL]
    lib.cmt_debug_buffer.argtypes = [VP, ctypes.c_char_p, fp, LL, llp]
    lib.cmt_get_stat.argtypes = [VP, ctypes.c_char_p, P(D), P(D)]
    lib.cmt_test_gemm.argtypes = [I, I, I, I, VP, LL, I, VP, LL, I, VP, LL, I, I, VP]
    U = ctypes.c_ulonglong
    lib.cmt_timeline.argtypes = [VP, ctypes.c_char_p, LL]
    lib.cmt_test_dropout.argtypes = [U, U, U, U, U, I, I, D, VP, VP, VP]
    _lib = lib
    return lib
