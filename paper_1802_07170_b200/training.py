"""Drop-in replacement for the reference train step.

``train_step(model, batch, cfg, lr, rng) -> float`` has the signature and
semantics of ``minmt.training.train_step`` (pkg/src/minmt/training.py:145-159):
it returns the label-smoothed loss, applies the clipped SGD update, leaves
parameter grads zero and advances ``rng`` by exactly the dropout draws the
reference consumes.  The work runs on the GPU engine; there is no CPU path.

Device parameters are authoritative between steps.  ``sync="eager"`` (the
default) copies the updated parameters back into ``model.params`` after
every step so callers see reference semantics; ``sync="lazy"`` skips that
and requires ``sync_to_host(model)`` before reading parameters (``install()``
wires these hooks into a reference ``Trainer``).
"""

from __future__ import annotations

import weakref

from .engine import DeviceSnapshot, Engine
from .errors import NumericError

_ENGINES: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
DEFAULTS = {"mode": "bf16", "sync": "eager", "device": 0}


def engine_for(model, mode=None, device=None):
    """The engine bound to ``model`` (created and uploaded on first use).  The
    model's ``ModelParams`` class gets the load_data / copy_data hooks
    (``_patch_params``) so host restores reach the device in every sync mode."""
    mode = mode or DEFAULTS["mode"]
    eng = _ENGINES.get(model)
    if eng is None or eng.mode != mode:
        eng = Engine(model.config, mode=mode, device=DEFAULTS["device"] if device is None else device)
        eng.upload(model.params)
        _ENGINES[model] = eng
        _patch_params(type(model.params))
    return eng


def sync_to_host(model):
    """Copy device parameters into ``model.params`` (before copy_data / save / dev_entropy)."""
    eng = _ENGINES.get(model)
    if eng is not None:
        eng.download_into(model.params)


def sync_from_host(model):
    """Re-upload ``model.params`` (after load_data / external edits)."""
    eng = _ENGINES.get(model)
    if eng is not None:
        eng.upload(model.params)


def train_step(model, batch, cfg, lr, rng, *, mode=None, sync=None):
    """One SGD update on a batch on the B200 engine; returns the smoothed loss.

    Frozen blocks (``ParamBlock.learnable`` False) are left out of the norm and
    the update (training.py:128-139).  When the gradient norm is not finite the
    reference raises before zeroing the grads (training.py:133-134, 141-142):
    the drop-in then leaves the step's gradients in the blocks' ``var.grad``
    too, with the weights unchanged."""
    eng = engine_for(model, mode)
    eng.set_learnable(model.params)
    try:
        loss, _ = eng.step(batch, lr, cfg.grad_clip_norm, cfg.label_smoothing, rng, update=True)
    except NumericError as e:
        if "gradient norm" in str(e):
            grads = eng.grads()
            for b in model.params.blocks():
                b.var.grad += grads[b.name].astype(b.var.grad.dtype)
        raise
    if (sync or DEFAULTS["sync"]) == "eager":
        eng.download_into(model.params)
    return loss


def dev_entropy(model, dev_batches, *, mode=None):
    """Drop-in for ``minmt.training.dev_entropy`` (training.py:162-182): mean
    per-token cross entropy (natural log), INFER mode, no label smoothing,
    computed by the device forward on the engine bound to ``model`` (device
    parameters are authoritative, so no host sync is needed)."""
    return engine_for(model, mode).dev_entropy(dev_batches)


def _engine_of(params):
    for m, eng in list(_ENGINES.items()):
        if m.params is params:
            return eng
    return None


def _patch_params(params_cls):
    """Wrap ``ModelParams.copy_data / load_data`` (model.py:104-115), once per class.

    * load_data (the Trainer's restore-from-best, training.py:254, 269) always
      reaches the device: a DeviceSnapshot of the bound engine is restored
      device to device, any other snapshot is loaded on the host as the
      reference does and then uploaded.  Without this, an eager-mode step
      after a host restore would train from the unrestored device weights.
    * copy_data (training.py:205, 246) returns a device-resident snapshot in
      lazy mode (a read-only name -> array mapping); in eager mode the host
      copy is current and the reference's own copy is returned.
    """
    if params_cls is None or getattr(params_cls, "_cmt_patched", False):
        return
    orig_load = params_cls.load_data
    orig_copy = params_cls.copy_data

    def copy_data(self):
        eng = _engine_of(self)
        if eng is not None and DEFAULTS["sync"] == "lazy":
            snap = eng.snapshot()
            if snap is not None:
                return snap
            eng.download_into(self)  # all slots in use: host copy of the device params
        return orig_copy(self)

    def load_data(self, snapshot):
        eng = _engine_of(self)
        if eng is not None and isinstance(snapshot, DeviceSnapshot) and snapshot.engine is eng:
            eng.restore(snapshot)  # device to device
            if DEFAULTS["sync"] == "eager":
                eng.download_into(self)
            return
        if isinstance(snapshot, DeviceSnapshot):
            snapshot = {n: snapshot[n] for n in snapshot}
        orig_load(self, snapshot)
        if eng is not None:
            eng.upload(self)

    params_cls.copy_data = copy_data
    params_cls.load_data = load_data
    params_cls._cmt_patched = True


def install(training_module=None, sync="lazy", params_cls=None):
    """Patch a reference ``minmt.training`` module to use this engine.

    ``Trainer.train`` resolves ``train_step`` and ``dev_entropy`` as module
    globals at call time (training.py:232, 243), so replacing them is
    sufficient for the step and the evaluation.  ``ModelParams.copy_data /
    load_data`` are wrapped (``_patch_params``) so the Trainer's snapshots and
    restore-from-best (training.py:205, 246-254, 269) stay on the device in
    lazy mode and reach it in eager mode.  With ``sync="lazy"``
    save_checkpoint first fetches the device parameters.
    """
    if training_module is None:
        import minmt.training as training_module  # type: ignore
    DEFAULTS["sync"] = sync
    training_module.train_step = train_step
    training_module.dev_entropy = dev_entropy  # device forward
    if sync == "lazy":
        orig_save = training_module.save_checkpoint

        def save_checkpoint(path, model, vocab_tokens):
            sync_to_host(model)
            return orig_save(path, model, vocab_tokens)

        training_module.save_checkpoint = save_checkpoint
    if params_cls is None:
        try:
            from minmt.model import ModelParams as params_cls  # type: ignore
        except Exception:
            params_cls = None
    _patch_params(params_cls)
    return training_module
