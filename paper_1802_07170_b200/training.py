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

_ENGINES: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
DEFAULTS = {"mode": "bf16", "sync": "eager", "device": 0}


def engine_for(model, mode=None, device=None):
    """The engine bound to ``model`` (created and uploaded on first use)."""
    mode = mode or DEFAULTS["mode"]
    eng = _ENGINES.get(model)
    if eng is None or eng.mode != mode:
        eng = Engine(model.config, mode=mode, device=DEFAULTS["device"] if device is None else device)
        eng.upload(model.params)
        _ENGINES[model] = eng
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
    """One SGD update on a batch on the B200 engine; returns the smoothed loss."""
    eng = engine_for(model, mode)
    loss, _ = eng.step(batch, lr, cfg.grad_clip_norm, cfg.label_smoothing, rng, update=True)
    if (sync or DEFAULTS["sync"]) == "eager":
        eng.download_into(model.params)
    return loss


def dev_entropy(model, dev_batches, *, mode=None):
    """Drop-in for ``minmt.training.dev_entropy`` (training.py:162-182): mean
    per-token cross entropy (natural log), INFER mode, no label smoothing,
    computed by the device forward on the engine bound to ``model`` (device
    parameters are authoritative, so no host sync is needed)."""
    return engine_for(model, mode).dev_entropy(dev_batches)


def install(training_module=None, sync="lazy", params_cls=None):
    """Patch a reference ``minmt.training`` module to use this engine.

    ``Trainer.train`` resolves ``train_step`` as a module global at call time
    (training.py:232), so replacing it is sufficient for the step.  With
    ``sync="lazy"`` the host-side readers of parameters are wrapped so the
    device copy is fetched first (save_checkpoint), ``ModelParams.copy_data``
    returns a device-resident snapshot (a read-only name -> array mapping) that
    ``ModelParams.load_data`` restores device-to-device (the Trainer's
    restore-from-best, training.py:205, 246-254, 269), and other host writes
    through ``load_data`` are pushed to the device.
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
        if params_cls is not None and not getattr(params_cls, "_cmt_patched", False):
            orig_load = params_cls.load_data
            orig_copy = params_cls.copy_data

            def _engine_of(params):
                for m, eng in list(_ENGINES.items()):
                    if m.params is params:
                        return eng
                return None

            def copy_data(self):
                # the Trainer keeps the best parameters (training.py:205, 246) and
                # hands them back to load_data: keep them on the device
                eng = _engine_of(self)
                if eng is not None:
                    snap = eng.snapshot()
                    if snap is not None:
                        return snap
                    eng.download_into(self)  # all slots in use: host copy of the device params
                return orig_copy(self)

            def load_data(self, snapshot):
                eng = _engine_of(self)
                if eng is not None and isinstance(snapshot, DeviceSnapshot) and snapshot.engine is eng:
                    eng.restore(snapshot)  # device to device (training.py:254, 269)
                    return
                orig_load(self, snapshot)
                if eng is not None:
                    eng.upload(self)

            params_cls.copy_data = copy_data
            params_cls.load_data = load_data
            params_cls._cmt_patched = True
    return training_module
