"""Python handle on one device engine (one model, one GPU).

Wraps the C ABI (include/cytonmt_b200.h) with numpy marshalling: parameter
upload/download by reference block name, batch staging, the step call, and
the PCG64 bookkeeping that keeps the caller's ``Rng`` in lock-step with the
reference (the device regenerates numpy's dropout draws bit-exactly; the
caller's generator is then advanced by the number of draws consumed).
"""

from __future__ import annotations

import ctypes
from collections.abc import Mapping

import numpy as np

from . import _lib
from .errors import ConfigError, MaskError, NumericError, ShapeError, ToolkitError

_ERRORS = {
    _lib.CMT_ERR_CONFIG: ConfigError,
    _lib.CMT_ERR_MASK: MaskError,
    _lib.CMT_ERR_SHAPE: ShapeError,
    _lib.CMT_ERR_NUM_SCORES: NumericError,
    _lib.CMT_ERR_NUM_LOGITS: NumericError,
    _lib.CMT_ERR_NUM_LOSS: NumericError,
    _lib.CMT_ERR_NUM_NORM: NumericError,
}
_NUMERIC_MSG = {
    _lib.CMT_ERR_NUM_SCORES: "softmax_columns received non-finite input",
    _lib.CMT_ERR_NUM_LOGITS: "log_softmax_columns received non-finite input",
    _lib.CMT_ERR_NUM_LOSS: "training loss is not finite",
    _lib.CMT_ERR_NUM_NORM: "gradient norm is not finite; step aborted",
}


def _fptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _llptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong))


def pcg_state(rng):
    """(state_hi, state_lo, inc_hi, inc_lo) of a reference Rng / numpy Generator."""
    gen = getattr(rng, "gen", rng)
    st = gen.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ConfigError(f"dropout parity needs a PCG64 generator, got {st.get('bit_generator')}")
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = (1 << 64) - 1
    return s >> 64, s & m, inc >> 64, inc & m


def dropout_draws(cfg, S, T, B):
    """Doubles the reference forward draws (SURVEY §3.1 order)."""
    if cfg.dropout <= 0.0:
        return 0
    L, H = cfg.depth, cfg.hidden_size
    return H * B * ((L - 1) * S + (L - 1) * T + T)


NSNAP = 4  # device snapshot slots (include/cytonmt_b200.h)


class DeviceSnapshot(Mapping):
    """Parameters saved on the device by Engine.snapshot().  Behaves like the
    reference's ``ModelParams.copy_data()`` dict (model.py:104-106): keys are
    the block names in registry order and ``snap[name]`` is an fp32 array (read
    from the device slot on first access).  ``Engine.restore`` / the installed
    ``ModelParams.load_data`` restore it without a host round trip."""

    def __init__(self, engine, slot):
        self.engine, self.slot, self.alive = engine, slot, True
        self._cache = {}

    def __getitem__(self, name):
        if name not in self._cache:
            eng = self.engine
            if not self.alive or eng.h is None:
                raise ConfigError("device snapshot was released")
            i = eng.index[name]
            out = np.empty(eng.blocks[i][1], dtype=np.float32)
            eng._check(eng.lib.cmt_snapshot_download(eng.h, self.slot, i, _fptr(out), out.shape[0], out.shape[1]))
            self._cache[name] = out
        return self._cache[name]

    def __iter__(self):
        return (n for n, _ in self.engine.blocks)

    def __len__(self):
        return len(self.engine.blocks)

    def release(self):
        if self.alive and getattr(self.engine, "h", None):
            self.engine.lib.cmt_snapshot_free(self.engine.h, self.slot)
        self.alive = False

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class Engine:
    def __init__(self, config, mode="bf16", device=0):
        self.lib = _lib.load()
        self.config = config
        self.mode = mode
        c = _lib.Config(int(config.vocab_size), int(config.embedding_size), int(config.hidden_size),
                        int(config.depth), int(bool(config.output_tanh)), int(bool(config.shared_embeddings)),
                        float(config.dropout), _lib.MODE_BF16 if mode == "bf16" else _lib.MODE_FP32)
        h = ctypes.c_void_p()
        rc = self.lib.cmt_create(ctypes.byref(c), int(device), ctypes.byref(h))
        if rc:
            raise self._exc(rc, self.lib.cmt_last_error(None))
        self.h = h
        self.blocks = []
        name = ctypes.create_string_buffer(256)
        r, cc = ctypes.c_longlong(), ctypes.c_longlong()
        for i in range(self.lib.cmt_num_blocks(h)):
            self._check(self.lib.cmt_block_info(h, i, name, 256, ctypes.byref(r), ctypes.byref(cc)))
            self.blocks.append((name.value.decode(), (r.value, cc.value)))
        self.index = {n: i for i, (n, _) in enumerate(self.blocks)}
        self.learnable = [True] * len(self.blocks)
        self.last_draws = 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.cmt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- errors ----
    @staticmethod
    def _exc(rc, msg):
        msg = msg.decode() if isinstance(msg, bytes) else str(msg)
        cls = _ERRORS.get(rc, RuntimeError if rc in (_lib.CMT_ERR_CUDA, _lib.CMT_ERR_INTERNAL) else ToolkitError)
        if rc in _NUMERIC_MSG:
            msg = _NUMERIC_MSG[rc]
        return cls(msg)

    def _check(self, rc):
        if rc:
            raise self._exc(rc, self.lib.cmt_last_error(self.h))

    # ---- parameters ----
    def upload(self, params):
        """params: reference ModelParams (blocks()) or {name: array}."""
        items = params.items() if isinstance(params, dict) else ((b.name, b.var.data) for b in params.blocks())
        seen = set()
        for n, arr in items:
            i = self.index[n]
            a = np.ascontiguousarray(arr, dtype=np.float32)
            if a.shape != self.blocks[i][1]:
                raise ShapeError(f"{n}: shape {a.shape} != {self.blocks[i][1]}")
            self._check(self.lib.cmt_upload_param(self.h, i, _fptr(a), a.shape[0], a.shape[1]))
            seen.add(n)
        missing = set(self.index) - seen
        if missing:
            raise ConfigError(f"upload is missing parameters {sorted(missing)}")

    def _download(self, fn, name):
        i = self.index[name]
        out = np.empty(self.blocks[i][1], dtype=np.float32)
        self._check(fn(self.h, i, _fptr(out), out.shape[0], out.shape[1]))
        return out

    def params(self):
        return {n: self._download(self.lib.cmt_download_param, n) for n, _ in self.blocks}

    def grads(self):
        return {n: self._download(self.lib.cmt_download_grad, n) for n, _ in self.blocks}

    # ---- device snapshots (ModelParams.copy_data / load_data, model.py:104-115) ----
    def snapshot(self):
        """Save the current parameters on the device; returns a DeviceSnapshot
        (a read-only {name: array} mapping that downloads blocks on access), or
        None when all snapshot slots are in use."""
        used = {sn.slot for sn in list(getattr(self, "_snaps", ())) if sn.alive}
        free = [i for i in range(NSNAP) if i not in used]
        if not free:
            return None
        sn = DeviceSnapshot(self, free[0])
        self._check(self.lib.cmt_snapshot_save(self.h, sn.slot))
        self._snaps = [x for x in getattr(self, "_snaps", ()) if x.alive] + [sn]
        return sn

    def restore(self, snap):
        """Load a DeviceSnapshot of this engine back into the parameters (device to device)."""
        if not isinstance(snap, DeviceSnapshot) or snap.engine is not self or not snap.alive:
            raise ConfigError("restore needs a live snapshot of this engine")
        self._check(self.lib.cmt_snapshot_restore(self.h, snap.slot))

    def set_learnable(self, flags):
        """{name: bool} or a reference ModelParams: frozen blocks (ParamBlock.learnable
        False, graph.py:20-31) are left out of the norm and the update
        (training.py:128-139)."""
        items = flags.items() if isinstance(flags, dict) else ((b.name, getattr(b, "learnable", True))
                                                                for b in flags.blocks())
        for n, on in items:
            i = self.index[n]
            if bool(on) != self.learnable[i]:
                self._check(self.lib.cmt_set_learnable(self.h, i, int(bool(on))))
                self.learnable[i] = bool(on)

    def download_into(self, params):
        for b in params.blocks():
            np.copyto(b.var.data, self._download(self.lib.cmt_download_param, b.name).astype(b.var.data.dtype))

    # ---- steps ----
    def stage(self, src_ids, src_mask, tgt_ids, tgt_mask):
        src = np.ascontiguousarray(src_ids, dtype=np.int64)
        tgt = np.ascontiguousarray(tgt_ids, dtype=np.int64)
        sm = np.ascontiguousarray(src_mask, dtype=np.float32)
        tm = np.ascontiguousarray(tgt_mask, dtype=np.float32)
        if src.ndim != 2 or tgt.ndim != 2 or src.shape[1] != tgt.shape[1] or sm.shape != src.shape \
                or tm.shape != tgt.shape:
            raise ShapeError(f"batch shapes disagree: src {src.shape} mask {sm.shape} tgt {tgt.shape} mask {tm.shape}")
        S, B = src.shape
        T = tgt.shape[0]
        self._staged = (src, sm, tgt, tm)  # keep host buffers alive for the call
        self._check(self.lib.cmt_stage_batch(self.h, _llptr(src), _fptr(sm), S, _llptr(tgt), _fptr(tm), T, B))
        self.shape = (S, T, B)

    def run(self, lr, clip, eps, rng=None, update=True, global_ntok=0.0, asynchronous=False, infer=False):
        """One step on the staged batch.  Advances ``rng`` by the draws used.
        ``infer=True``: forward only in INFER mode (no dropout/backward/update)."""
        st = pcg_state(rng) if rng is not None else (0, 0, 0, 1)
        a = _lib.StepArgs(float(lr), float(clip) if clip is not None else float("nan"), float(eps),
                          st[0], st[1], st[2], st[3], float(global_ntok),
                          (0 if update else _lib.FLAG_NO_UPDATE) | (_lib.FLAG_ASYNC if asynchronous else 0)
                          | (_lib.FLAG_INFER if infer else 0))
        r = _lib.StepResult()
        rc = self.lib.cmt_run_step(self.h, ctypes.byref(a), ctypes.byref(r))
        self.last_draws = r.draws
        if rng is not None and r.draws and rc in (0, _lib.CMT_ERR_NUM_SCORES, _lib.CMT_ERR_NUM_LOGITS,
                                                    _lib.CMT_ERR_NUM_LOSS, _lib.CMT_ERR_NUM_NORM):
            getattr(rng, "gen", rng).bit_generator.advance(int(r.draws))
        self._check(rc)
        return r

    def wait(self):
        r = _lib.StepResult()
        self._check(self.lib.cmt_wait(self.h, ctypes.byref(r)))
        return r

    def _stage_batch(self, batch, rng):
        src, tgt = batch.src_ids, batch.tgt_ids
        try:
            self.stage(src, batch.src_mask, tgt, batch.tgt_mask)
            if getattr(self, "_dp", None) is not None:
                from . import dp
                dp.exchange_rows(self, self._dp)
        except ConfigError as e:
            # the reference raises the empty-target ConfigError after its forward
            # pass, so the dropout draws are consumed (training.py:149-153)
            if "unmasked token" in str(e) and rng is not None:
                S, B = np.shape(src)
                n = dropout_draws(self.config, S, np.shape(tgt)[0], B)
                if n:
                    getattr(rng, "gen", rng).bit_generator.advance(n)
            raise

    def step(self, batch, lr, clip, eps, rng=None, update=True):
        """Stage + run: returns (loss, grad_norm)."""
        self._stage_batch(batch, rng)
        r = self.run(lr, clip, eps, rng, update)
        return r.loss, r.grad_norm

    def pipeline(self, batches, lr, clip, eps, rng=None, global_ntok=0.0):
        """Train on ``batches`` in order, yielding (loss, grad_norm) per batch.

        Same results as calling ``step`` per batch (same updates, same draws),
        but batch i+1 is validated, converted, segment-sorted and copied into
        pinned memory on the host while step i still runs on the device (the
        staging buffers are double-buffered); step i's result is read back
        before step i+1 is launched.  A NumericError of step i is raised when
        its result is collected (the device already skipped its update)."""
        pending = False
        for batch in batches:
            try:
                self._stage_batch(batch, rng)
            except Exception:
                if pending:
                    pending = False
                    yield self._finish()
                raise
            if pending:
                pending = False
                yield self._finish()
            self.run(lr, clip, eps, rng, asynchronous=True, global_ntok=global_ntok)
            pending = True
        if pending:
            yield self._finish()

    # ---- translation: batched beam search on the device (cmt_beam_*, include/cytonmt_b200.h) ----
    def beam_search(self, sources, beam, n_best, max_lens, lp_table, steps_per_call=16):
        """Beam search for a list of non-empty id sequences at once.

        ``max_lens[i]`` is sentence i's length cap, ``lp_table[n]`` the length
        penalty of n tokens.  Returns, per sentence, the list of results
        ``(tokens, score, log_prob, truncated)`` (score None when truncated)."""
        B = len(sources)
        S = max(len(x) for x in sources)
        src = np.zeros((S, B), dtype=np.int64)
        mask = np.zeros((S, B), dtype=np.float32)
        for b, x in enumerate(sources):
            src[:len(x), b] = np.asarray(x, dtype=np.int64)
            mask[:len(x), b] = 1.0
        ml = np.ascontiguousarray(max_lens, dtype=np.int32)
        lpt = np.ascontiguousarray(lp_table, dtype=np.float64)
        ip = ctypes.POINTER(ctypes.c_int)
        dp = ctypes.POINTER(ctypes.c_double)
        self._check(self.lib.cmt_beam_begin(self.h, _llptr(src), _fptr(mask), S, B, int(beam), int(n_best),
                                            ml.ctypes.data_as(ip), lpt.ctypes.data_as(dp), int(lpt.size)))
        active = ctypes.c_int(1)
        while active.value:
            self._check(self.lib.cmt_beam_step(self.h, int(steps_per_call), ctypes.byref(active)))
        cap = int(ml.max()) + 1
        toks = np.empty(cap, dtype=np.int32)
        n_tok, n_res, trunc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        score, logp = ctypes.c_double(), ctypes.c_double()
        out = []
        for b in range(B):
            res, rank = [], 0
            while True:
                self._check(self.lib.cmt_beam_result(self.h, b, rank, toks.ctypes.data_as(ip), cap, ctypes.byref(n_tok),
                                                     ctypes.byref(score), ctypes.byref(logp), ctypes.byref(trunc),
                                                     ctypes.byref(n_res)))
                res.append(([int(t) for t in toks[:n_tok.value]], None if trunc.value else score.value, logp.value,
                            bool(trunc.value)))
                rank += 1
                if rank >= n_res.value:
                    break
            out.append(res)
        return out

    def _finish(self):
        r = self.wait()
        return r.loss, r.grad_norm

    def dev_entropy(self, batches):
        """Mean per-token cross entropy over ``batches`` in INFER mode, no label
        smoothing (reference training.py:162-182); every batch runs the device
        forward, only the per-batch loss sum and token count come back."""
        if not batches:
            raise ConfigError("development set is empty")
        total, tokens = 0.0, 0.0
        self.set_option("allow_empty_targets", 1)
        try:
            for batch in batches:
                self.stage(batch.src_ids, batch.src_mask, batch.tgt_ids, batch.tgt_mask)
                r = self.run(0.0, None, 0.0, None, update=False, infer=True)
                total += float(r.loss_sum)
                tokens += float(r.ntok)
        finally:
            self.set_option("allow_empty_targets", 0)
        return total / tokens

    def debug_buffer(self, name, cap=1 << 28):
        out = np.empty(cap, dtype=np.float32)
        n = ctypes.c_longlong()
        self._check(self.lib.cmt_debug_buffer(self.h, name.encode(), _fptr(out), cap, ctypes.byref(n)))
        return out[:n.value].copy()

    # ---- data parallel ----
    def set_dp(self, dist, rank, world):
        from . import dp
        dp.attach(self, dist, rank, world)
        self._dp = dist if world > 1 else None

    @property
    def n_tables(self):
        return 1 if self.config.shared_embeddings else 2

    def staged_rows(self, table):
        """Ascending ids of embedding table ``table`` the staged batch touches."""
        n = ctypes.c_int()
        self._check(self.lib.cmt_staged_rows(self.h, int(table), None, 0, ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.int32)
        self._check(self.lib.cmt_staged_rows(self.h, int(table), out.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                             n.value, ctypes.byref(n)))
        return out

    def set_union(self, table, ids):
        """Rows union (ascending ids over all ranks) of table ``table`` for the next step."""
        u = np.ascontiguousarray(ids, dtype=np.int32)
        self._check(self.lib.cmt_set_union(self.h, int(table), u.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                           int(u.size)))

    # ---- timing ----
    def set_option(self, key, value):
        self._check(self.lib.cmt_set_option(self.h, key.encode(), int(value)))

    def timeline(self, cap=1 << 22):
        """[(label, ms)] per launch since set_option("timeline", 1) (debug)."""
        buf = ctypes.create_string_buffer(cap)
        self._check(self.lib.cmt_timeline(self.h, buf, cap))
        out = []
        for line in buf.value.decode().splitlines():
            lab, ms = line.rsplit("\t", 1)
            out.append((lab, float(ms)))
        return out

    def stat(self, key):
        v, c = ctypes.c_double(), ctypes.c_double()
        self._check(self.lib.cmt_get_stat(self.h, key.encode(), ctypes.byref(v), ctypes.byref(c)))
        return v.value, c.value

    def record(self, slot):
        self._check(self.lib.cmt_event_record(self.h, slot))

    def elapsed_ms(self, a, b):
        ms = ctypes.c_float()
        self._check(self.lib.cmt_event_elapsed(self.h, a, b, ctypes.byref(ms)))
        return ms.value


def launch_count():
    return _lib.load().cmt_launch_count()
