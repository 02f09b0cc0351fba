"""CPU oracle for the CytonMT/minmt train step — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``--impl reference`` and ``cpu_baseline``) may import it.  The CUDA engine in
``paper_1802_07170_b200`` never routes through it.

It is a functional numpy restatement of the reference's teacher-forced
forward + backward + clipped-SGD step.  The reference builds a per-batch
``LayerChain`` of ``Layer`` objects (``/root/reference/pkg/src/minmt/model.py:267-327``);
here the same math is written as plain functions over a ``{block name: array}``
dict so each equation can be checked against the file:line it follows:

* embedding gather / scatter-add ............ tensor.py:191-216, layers.py:79-113
* LSTM cell forward / backward .............. layers.py:344-395
* masked (optionally reversed) LSTM scan .... layers.py:404-503
* bidirectional first encoder layer (SUM) ... model.py:285-292, layers.py:162-180
* dropout (inverted, PCG64 draws) ........... layers.py:265-296
* Luong "general" attention chain ........... attention.py:46-84, 139-173, layers.py:183-215
* output projection (+tanh) ................. model.py:311-314, layers.py:32-76
* log-softmax + label-smoothed CE ........... tensor.py:146-151, training.py:96-120
* global-norm clip + SGD .................... training.py:123-142
* the step itself ........................... training.py:145-159

Layout follows the reference: activations are ``(dim, steps*batch)`` with
column ``n = t*B + b``; id matrices are ``(steps, batch)``.

Parity is PINNED: ``tests/golden/make_golden.py`` runs the real reference
(imported from /root/reference in the authoring container) on seeded inputs
and commits its loss, gradients and updated weights; ``tests/test_oracle.py``
checks this module against those fixtures at fp32 (and fp64) tolerance.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

BOS, EOS, PAD = 2, 3, 0
GATES = ("i", "f", "g", "o")
MASK_FILL = -1e9  # additive attention mask, layers.py:190


class OracleError(Exception):
    """Raised where the reference raises one of its ToolkitError subclasses."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind  # "ConfigError" | "MaskError" | "NumericError" | "ShapeError"


# ---------------------------------------------------------------------------
# Parameter registry (model.py:65-115): names, shapes, init order
# ---------------------------------------------------------------------------

@dataclass
class Dims:
    vocab: int
    emb: int
    hidden: int
    depth: int
    dropout: float = 0.2
    output_tanh: bool = True
    shared_embeddings: bool = False


def lstm_names(prefix: str):
    return [f"{prefix}.w_{g}" for g in GATES] + [f"{prefix}.b_{g}" for g in GATES]


def registry(d: Dims):
    """[(name, shape)] in the reference's declaration order (model.py:86-95)."""
    V, E, H, L = d.vocab, d.emb, d.hidden, d.depth
    out = [("src_embed", (V, E))]
    if not d.shared_embeddings:
        out.append(("tgt_embed", (V, E)))

    def lstm(prefix, din):
        return [(f"{prefix}.w_{g}", (din + H, H)) for g in GATES] + \
               [(f"{prefix}.b_{g}", (H, 1)) for g in GATES]

    out += lstm("enc.l1.fwd", E) + lstm("enc.l1.bwd", E)
    for k in range(2, L + 1):
        out += lstm(f"enc.l{k}", H)
    for k in range(1, L + 1):
        out += lstm(f"dec.l{k}", E if k == 1 else H)
    out += [("att.w_a.w", (H, H)), ("att.w_c.w", (2 * H, H)), ("out.w", (H, V)), ("out.b", (V, 1))]
    return out


def init_params(d: Dims, gen: np.random.Generator, dtype=np.float32):
    """Uniform(+-0.1) weights, zero biases, forget bias 1.0.

    Draw order = construction order (model.py:73-85, layers.py:37-38, 313-321):
    every weight matrix draws gen.uniform in registry order; biases draw
    nothing.  The tgt table draws after src unless shared.
    """
    p = {}
    for name, shape in registry(d):
        if name.endswith(".b_i") or name.endswith(".b_f") or name.endswith(".b_g") \
                or name.endswith(".b_o") or name == "out.b":
            p[name] = np.zeros(shape, dtype=dtype)
            if name.endswith(".b_f"):
                p[name].fill(1.0)
        else:
            p[name] = gen.uniform(-0.1, 0.1, size=shape).astype(dtype)
    return p


# ---------------------------------------------------------------------------
# Pointwise kernels (tensor.py:157-176)
# ---------------------------------------------------------------------------

def sigmoid(x):
    # branch-split stable form (tensor.py:165-172)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def log_softmax_cols(x):
    """tensor.py:146-151 (raises on non-finite input)."""
    if not np.all(np.isfinite(x)):
        raise OracleError("NumericError", "log_softmax_columns received non-finite input")
    s = x - x.max(axis=0, keepdims=True)
    return s - np.log(np.exp(s).sum(axis=0, keepdims=True))


def softmax_cols(x):
    """tensor.py:137-143."""
    if not np.all(np.isfinite(x)):
        raise OracleError("NumericError", "softmax_columns received non-finite input")
    e = np.exp(x - x.max(axis=0, keepdims=True))
    return e / e.sum(axis=0, keepdims=True)


# ---------------------------------------------------------------------------
# LSTM (layers.py:344-503)
# ---------------------------------------------------------------------------

def _lstm_w(p, prefix):
    return [p[f"{prefix}.w_{g}"] for g in GATES], [p[f"{prefix}.b_{g}"] for g in GATES]


def lstm_scan(p, prefix, x, steps, batch, mask=None, reverse=False, h0=None, c0=None):
    """Masked LSTM scan, layers.py:440-467 with the cell of layers.py:344-363.

    x is (Din, steps*batch).  Padded steps (mask 0) carry (h, c) through.
    Returns y (H, steps*batch), final (h, c) and a per-step cache.
    """
    W, bias = _lstm_w(p, prefix)
    H = W[0].shape[1]
    din = x.shape[0]
    dt = x.dtype
    x3 = x.reshape(din, steps, batch)
    y = np.zeros((H, steps * batch), dtype=dt)
    y3 = y.reshape(H, steps, batch)
    h = np.zeros((H, batch), dt) if h0 is None else h0.copy()
    c = np.zeros((H, batch), dt) if c0 is None else c0.copy()
    cache = []
    order = range(steps - 1, -1, -1) if reverse else range(steps)
    for t in order:
        z = np.concatenate([x3[:, t, :], h], axis=0)
        a = {}
        for gi, g in enumerate(GATES):
            u = W[gi].T @ z + bias[gi]
            a[g] = np.tanh(u) if g == "g" else sigmoid(u)
        c_new = a["f"] * c + a["i"] * a["g"]
        tc = np.tanh(c_new)
        h_new = a["o"] * tc
        if mask is not None:
            m = mask[t][np.newaxis, :].astype(dt)
            h_next = m * h_new + (1.0 - m) * h
            c_next = m * c_new + (1.0 - m) * c
        else:
            m = None
            h_next, c_next = h_new, c_new
        cache.append((t, z, a, c, tc, m))
        y3[:, t, :] = h_next
        h, c = h_next, c_next
    return y, (h, c), cache


def lstm_scan_backward(p, prefix, grads, dy, cache, din, steps, batch, dh_final, dc_final):
    """BPTT, layers.py:469-493 with the cell backward of layers.py:366-395.

    Accumulates weight/bias grads into ``grads`` (per-step, as the reference
    does at layers.py:389-391) and returns (dx, dh_init, dc_init).
    """
    W, _ = _lstm_w(p, prefix)
    H = W[0].shape[1]
    dt = dy.dtype
    dy3 = dy.reshape(H, steps, batch)
    dx = np.zeros((din, steps * batch), dtype=dt)
    dx3 = dx.reshape(din, steps, batch)
    dh = dh_final.copy()
    dc = dc_final.copy()
    gw = [grads[f"{prefix}.w_{g}"] for g in GATES]
    gb = [grads[f"{prefix}.b_{g}"] for g in GATES]
    for t, z, a, c_prev, tc, m in reversed(cache):
        dh = dh + dy3[:, t, :]
        if m is not None:
            dh_new, dc_new = m * dh, m * dc
            dh_carry, dc_carry = (1.0 - m) * dh, (1.0 - m) * dc
        else:
            dh_new, dc_new = dh, dc
            dh_carry = dc_carry = 0.0
        i, f, g, o = a["i"], a["f"], a["g"], a["o"]
        dc_tot = dh_new * o * (1.0 - tc * tc) + dc_new
        du = [dc_tot * g * (i * (1.0 - i)),
              dc_tot * c_prev * (f * (1.0 - f)),
              dc_tot * i * (1.0 - g * g),
              dh_new * tc * (o * (1.0 - o))]
        dz = np.zeros_like(z)
        for k in range(4):
            dz += W[k] @ du[k]
            gw[k] += z @ du[k].T
            gb[k] += du[k].sum(axis=1, keepdims=True)
        dx3[:, t, :] += dz[:din]
        dh = dz[din:] + dh_carry
        dc = dc_tot * f + dc_carry
    return dx, dh, dc


# ---------------------------------------------------------------------------
# Dropout (layers.py:265-296): one gen.random(shape) draw per site, C order
# ---------------------------------------------------------------------------

def dropout_mask(shape, rate, gen, dtype):
    if rate <= 0.0:
        return None
    keep = gen.random(size=shape) >= rate
    return keep.astype(dtype) / (1.0 - rate)


def dropout_draws(d: Dims, S: int, T: int, B: int) -> int:
    """Number of doubles the train-mode forward draws (SURVEY §3.1 order)."""
    if d.dropout <= 0.0:
        return 0
    return d.hidden * B * ((d.depth - 1) * S + (d.depth - 1) * T + T)


# ---------------------------------------------------------------------------
# Attention (attention.py:46-84, 139-173)
# ---------------------------------------------------------------------------

def attention_forward(wa, wc, hs, ht, S, T, B, src_mask):
    H = hs.shape[0]
    hs3 = hs.reshape(H, S, B)
    u = wa.T @ ht                                         # Linear(W_a), :166
    u3 = u.reshape(H, T, B)
    scores = np.einsum("hsb,hqb->sqb", hs3, u3).reshape(S, T * B)
    full = np.broadcast_to(src_mask[:, None, :], (S, T, B)).reshape(S, T * B)
    additive = ((1.0 - full) * MASK_FILL).astype(hs.dtype)
    alpha = softmax_cols(scores + additive)               # layers.py:206-208
    a3 = alpha.reshape(S, T, B)
    ctx = np.einsum("hsb,sqb->hqb", hs3, a3).reshape(H, T * B)
    cst = np.concatenate([ctx, ht], axis=0)               # :170
    ho = np.tanh(wc.T @ cst)                              # :171-172
    return dict(u=u, alpha=alpha, ctx=ctx, cst=cst, ho=ho)


def attention_backward(wa, wc, hs, ht, S, T, B, fw, dho, grads):
    H = hs.shape[0]
    hs3 = hs.reshape(H, S, B)
    dpre = dho * (1.0 - fw["ho"] * fw["ho"])
    dcst = wc @ dpre
    grads["att.w_c.w"] += fw["cst"] @ dpre.T
    dctx, dht = dcst[:H], dcst[H:].copy()
    a3 = fw["alpha"].reshape(S, T, B)
    d3 = dctx.reshape(H, T, B)
    dhs = np.einsum("hqb,sqb->hsb", d3, a3)
    dalpha = np.einsum("hsb,hqb->sqb", hs3, d3).reshape(S, T * B)
    p = fw["alpha"]
    dscores = p * (dalpha - (p * dalpha).sum(axis=0, keepdims=True))
    u3 = fw["u"].reshape(H, T, B)
    ds3 = dscores.reshape(S, T, B)
    dhs += np.einsum("hqb,sqb->hsb", u3, ds3)
    du = np.einsum("hsb,sqb->hqb", hs3, ds3).reshape(H, T * B)
    dht += wa @ du
    grads["att.w_a.w"] += ht @ du.T
    return dhs.reshape(H, S * B), dht


# ---------------------------------------------------------------------------
# Loss (training.py:96-120)
# ---------------------------------------------------------------------------

def smoothed_loss(lp, targets, eps, mask):
    V, n = lp.shape
    mask = np.ones(n, lp.dtype) if mask is None else np.asarray(mask, lp.dtype)
    ntok = mask.sum()
    if ntok <= 0:
        raise OracleError("ConfigError", "smoothed_loss needs at least one unmasked token")
    cols = np.arange(n)
    per_tok = -((1.0 - eps) * lp[targets, cols] + (eps / V) * lp.sum(axis=0))
    loss = float((per_tok * mask).sum() / ntok)
    d = np.exp(lp)
    d[targets, cols] -= 1.0 - eps
    d -= eps / V
    d *= mask[np.newaxis, :] / ntok
    return loss, d


# ---------------------------------------------------------------------------
# The step
# ---------------------------------------------------------------------------

def check_ids(ids, V):
    """model.py:146-151."""
    ids = np.asarray(ids, dtype=np.int64)
    if ids.size and (ids.min() < 0 or ids.max() >= V):
        bad = ids[(ids < 0) | (ids >= V)][0]
        raise OracleError("ConfigError", f"token id {int(bad)} outside vocabulary of size {V}")
    return ids


def shift_targets(tgt, bos=BOS):
    """model.py:239-244."""
    out = np.empty_like(tgt)
    out[0] = bos
    out[1:] = tgt[:-1]
    return out


def forward_backward(p, d: Dims, src_ids, src_mask, tgt_ids, tgt_mask, eps, gen=None,
                     masks=None, want_grads=True):
    """Loss and per-block gradients of one teacher-forced batch.

    ``gen`` supplies dropout draws (numpy Generator, reference draw order);
    alternatively ``masks`` is a list of precomputed dropout masks in draw
    order (None entries = identity).  Returns (loss, grads, aux).
    """
    dt = p["src_embed"].dtype
    V, H, L = d.vocab, d.hidden, d.depth
    src_ids = check_ids(src_ids, V)
    tgt_in = check_ids(shift_targets(np.asarray(tgt_ids, np.int64)), V)
    S, B = src_ids.shape
    T = tgt_in.shape[0]
    src_mask = np.asarray(src_mask, dtype=dt)
    if not (src_mask > 0).any(axis=0).all():
        raise OracleError("MaskError", "a batch column has every source position masked")
    tgt_embed = "src_embed" if d.shared_embeddings else "tgt_embed"

    mask_iter = iter(masks) if masks is not None else None

    def next_mask(shape):
        if mask_iter is not None:
            return next(mask_iter)
        return dropout_mask(shape, d.dropout, gen, dt)

    # ---- encoder (model.py:285-297)
    xs = p["src_embed"][src_ids.reshape(-1)].T.copy()
    yf, _, cf = lstm_scan(p, "enc.l1.fwd", xs, S, B, mask=src_mask)
    yb, (hb, cb), cb_ = lstm_scan(p, "enc.l1.bwd", xs, S, B, mask=src_mask, reverse=True)
    top = yf + yb
    finals = [(hb, cb)]
    enc_layers = []  # (prefix, input, mask_drop, cache)
    for k in range(2, L + 1):
        md = next_mask(top.shape)
        inp = top if md is None else top * md
        y, fin, cache = lstm_scan(p, f"enc.l{k}", inp, S, B, mask=src_mask)
        enc_layers.append((f"enc.l{k}", inp, md, cache))
        finals.append(fin)
        top = y
    hs = top

    # ---- decoder (model.py:299-306), unmasked, init from encoder finals
    x = p[tgt_embed][tgt_in.reshape(-1)].T.copy()
    dec_layers = []
    for k in range(1, L + 1):
        md = None
        if k > 1:
            md = next_mask(x.shape)
            if md is not None:
                x = x * md
        y, _, cache = lstm_scan(p, f"dec.l{k}", x, T, B, h0=finals[k - 1][0], c0=finals[k - 1][1])
        dec_layers.append((f"dec.l{k}", x.shape[0], md, cache))
        x = y
    ht = x

    # ---- attention + output (model.py:308-314)
    fw = attention_forward(p["att.w_a.w"], p["att.w_c.w"], hs, ht, S, T, B, src_mask)
    mo = next_mask(fw["ho"].shape)
    hod = fw["ho"] if mo is None else fw["ho"] * mo
    logits = p["out.w"].T @ hod + p["out.b"]
    if d.output_tanh:
        logits = np.tanh(logits)

    # ---- loss (training.py:149-155)
    lp = log_softmax_cols(logits)
    loss, dlogits = smoothed_loss(lp, np.asarray(tgt_ids, np.int64).reshape(T * B), eps,
                                  np.asarray(tgt_mask).reshape(T * B))
    if not math.isfinite(loss):
        raise OracleError("NumericError", f"training loss is not finite: {loss}")
    aux = dict(logits=logits, hs=hs, ht=ht, alpha=fw["alpha"], ho=fw["ho"])
    if not want_grads:
        return loss, None, aux

    # ---- backward
    g = {name: np.zeros(shape, dtype=dt) for name, shape in registry(d)}
    dlogits = dlogits.astype(dt)
    dpre = dlogits * (1.0 - logits * logits) if d.output_tanh else dlogits
    g["out.w"] += hod @ dpre.T
    g["out.b"] += dpre.sum(axis=1, keepdims=True)
    dhod = p["out.w"] @ dpre
    dho = dhod if mo is None else dhod * mo
    dhs, dht = attention_backward(p["att.w_a.w"], p["att.w_c.w"], hs, ht, S, T, B, fw, dho, g)

    # decoder BPTT, top layer first; init-state grads flow to encoder finals
    dfinal = [None] * L
    dy = dht
    for k in range(L, 0, -1):
        prefix, din, md, cache = dec_layers[k - 1]
        zero = np.zeros((H, B), dt)
        dx, dh0, dc0 = lstm_scan_backward(p, prefix, g, dy, cache, din, T, B, zero, zero)
        dfinal[k - 1] = (dh0, dc0)
        dy = dx if md is None else dx * md
    dtgt_x = dy
    np.add.at(g[tgt_embed], tgt_in.reshape(-1), dtgt_x.T)

    # encoder deep layers, top first
    dtop = dhs
    for k in range(L, 1, -1):
        prefix, inp, md, cache = enc_layers[k - 2]
        dx, _, _ = lstm_scan_backward(p, prefix, g, dtop, cache, H, S, B, dfinal[k - 1][0], dfinal[k - 1][1])
        dtop = dx if md is None else dx * md
    # layer 1: the sum feeds both directions; decoder l1 init came from the bwd final
    zero = np.zeros((H, B), dt)
    E = d.emb
    dxb, _, _ = lstm_scan_backward(p, "enc.l1.bwd", g, dtop, cb_, E, S, B, dfinal[0][0], dfinal[0][1])
    dxf, _, _ = lstm_scan_backward(p, "enc.l1.fwd", g, dtop, cf, E, S, B, zero, zero)
    np.add.at(g["src_embed"], src_ids.reshape(-1), (dxf + dxb).T)
    return loss, g, aux


def dev_entropy(p, d: Dims, batches):
    """Mean per-token natural-log cross entropy, inference mode, no smoothing
    (reference training.py:162-182): sum over batches of -(lp_gold * m) in
    fp32, divided by the token count."""
    if not batches:
        raise OracleError("ConfigError", "development set is empty")
    total, tokens = 0.0, 0.0
    nmask = 2 * (d.depth - 1) + 1
    for src, sm, tgt, tm in batches:
        # identity dropout masks = INFER mode (layers.py:283-290)
        _, _, aux = forward_backward(p, d, src, sm, tgt, np.ones_like(np.asarray(tm, np.float32)), 0.0,
                                     masks=[None] * nmask, want_grads=False)
        lp = log_softmax_cols(aux["logits"])
        T, B = np.asarray(tgt).shape
        gold = lp[np.asarray(tgt, np.int64).reshape(T * B), np.arange(T * B)]
        m = np.asarray(tm, np.float32).reshape(T * B)
        total += float(-(gold * m).sum())
        tokens += float(m.sum())
    return total / tokens


def sgd_step(p, g, names, lr, clip):
    """training.py:123-142: global L2 norm (fp32 dots summed in double), clip, update.

    Raises NumericError (no update) on a non-finite norm.  Returns the norm.
    """
    sq = 0.0
    for n in names:
        gv = g[n].ravel()
        sq += float(np.dot(gv, gv))
    norm = math.sqrt(sq)
    if not math.isfinite(norm):
        raise OracleError("NumericError", "gradient norm is not finite; step aborted")
    scale = 1.0
    if clip is not None and norm > clip:
        scale = clip / norm
    for n in names:
        p[n] -= (lr * scale) * g[n]
    return norm


def train_step(p, d: Dims, batch, eps, lr, clip, gen):
    """training.py:145-159 on a param dict.  Returns (loss, grad_norm, grads)."""
    src_ids, src_mask, tgt_ids, tgt_mask = batch
    loss, g, _ = forward_backward(p, d, src_ids, src_mask, tgt_ids, tgt_mask, eps, gen=gen)
    norm = sgd_step(p, g, [n for n, _ in registry(d)], lr, clip)
    return loss, norm, g


# ---------------------------------------------------------------------------
# Synthetic batches
# ---------------------------------------------------------------------------

def synthetic_batch(V, S, T, B, seed=0, ragged=False):
    """ids uniform in [4, V); last target row EOS; masks all ones.

    ``ragged``: alternate columns lose their last k source/target positions
    (PAD=0, mask 0); the target gets EOS at the sentence end.
    """
    g = np.random.default_rng(seed)
    src = g.integers(4, V, (S, B)).astype(np.int64)
    tgt = g.integers(4, V, (T, B)).astype(np.int64)
    tgt[T - 1, :] = EOS
    sm = np.ones((S, B), np.float32)
    tm = np.ones((T, B), np.float32)
    if ragged:
        for b in range(1, B, 2):
            ks = 1 + (b // 2) % max(1, S - 1)
            kt = 1 + (b // 2) % max(1, T - 1)
            src[S - ks:, b] = PAD
            sm[S - ks:, b] = 0.0
            tgt[T - kt - 1, b] = EOS
            tgt[T - kt:, b] = PAD
            tm[T - kt:, b] = 0.0
    return src, sm, tgt, tm


def norm_rel_err(a, r):
    """max|a-r| / max(|a|inf, |r|inf) — pkg/tests/helpers.py:80-81."""
    a = np.asarray(a, np.float64)
    r = np.asarray(r, np.float64)
    scale = max(np.abs(a).max(initial=0.0), np.abs(r).max(initial=0.0), 1e-30)
    return float(np.abs(a - r).max(initial=0.0) / scale)
