"""Shared helpers for the GPU parity tests (engine vs golden fixtures / oracle)."""

import numpy as np

from oracle import minmt_oracle as O
from paper_1802_07170_b200.engine import Engine
from paper_1802_07170_b200.model import Batch, ModelConfig


def cfg_of(d: O.Dims):
    return ModelConfig(d.vocab, d.emb, d.hidden, d.depth, d.dropout, d.output_tanh, d.shared_embeddings)


def engine_step(d, params, batch, eps, lr, clip, seed, mode, update=True):
    """Run the CUDA engine on (params, batch).  Returns loss, norm, grads (if
    not update), new params, the advanced numpy generator."""
    eng = Engine(cfg_of(d), mode=mode)
    eng.upload(params)
    gen = np.random.Generator(np.random.PCG64(seed))
    src, sm, tgt, tm = batch
    loss, norm = eng.step(Batch(src, tgt, sm, tm), lr, clip, eps, gen, update=update)
    grads = None if update else eng.grads()
    newp = eng.params()
    eng.close()
    return loss, norm, grads, newp, gen


def oracle_step(d, params, batch, eps, lr, clip, seed, update=True):
    p = {k: v.copy() for k, v in params.items()}
    gen = np.random.Generator(np.random.PCG64(seed))
    src, sm, tgt, tm = batch
    loss, g, _ = O.forward_backward(p, d, src, sm, tgt, tm, eps, gen=gen)
    norm = None
    if update:
        norm = O.sgd_step(p, g, [n for n, _ in O.registry(d)], lr, clip)
    return loss, norm, g, p, gen


def scaled_params(d, seed, scale):
    gen = np.random.Generator(np.random.PCG64(seed))
    return {n: gen.uniform(-scale, scale, size=s).astype(np.float32) for n, s in O.registry(d)}


def step_close(new, old, ref_new, rel):
    """The applied step w_new - w_old against the reference's, to `rel` of the
    step's size plus one fp32 ulp of the weights: w - fp32(s*g) rounds to fp32,
    so grads equal to ~1e-5 can still land one ulp apart, and one ulp of a 0.1
    weight is ~1e-3 of a 1e-5 step."""
    new, old, ref_new = (np.asarray(x, np.float64) for x in (new, old, ref_new))
    ulp = float(np.spacing(np.float32(np.abs(ref_new).max())))
    err = float(np.abs(new - ref_new).max())
    return err <= rel * float(np.abs(ref_new - old).max()) + ulp, err
