"""CPU oracle of the neural GPUMemNet ensemble — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module, and only as the checker; the product path
(libcarma_b200.so, carma_nn_*) never calls it.

What it restates. The paper's GPUMemNet ensembles: the
Transformer ensemble (tf_logits) and the MLP ensemble (fig. "MLP Ensemble"): each member is a stack of ReLU layers with batch norm
(folded into the linear layers at export), a linear head over the memory
bins, a softmax; the ensemble averages the members' probabilities and the
predicted bin is the argmax (ties to the larger bin, the vote rule of
estimators.cpp:463-474); bytes = (bin + 1) * range (estimate_learned,
estimators.cpp:540-551). Features are scalar_features
(estimators.cpp:317-342) under the input transform documented in
include/carma_gpu.h.

Parity status: the reference artifact has NO neural estimator (SURVEY.md F1,
§8(f)4), so this oracle cannot be pinned to reference outputs. It is pinned
instead to the PyTorch model that defines the weights: tests/golden/
gpumemnet.npz holds the torch fp64 forward pass (eval mode, batch norm
folded, bf16-rounded weights) of scripts/train_gpumemnet.py on fixed rows,
and tests/test_gpumemnet.py checks this oracle against it.

Arithmetic: the input transform as the kernel (fp32; log1p within an ulp or
two of CUDA's log1pf); layers, softmax and the mean in fp64.
"""
from __future__ import annotations

import numpy as np

DIMS = 19


def unpack_params(spec, params: np.ndarray):
    """[(layers[(W, b)], (W_head, b_head))] per member from the flat layout of
    carma_nn_set_model (carma_gpu.h)."""
    members = []
    at = 0
    for e in range(int(spec["members"])):
        layers = []
        fan_in = DIMS
        for l in range(int(spec["depth"][e])):
            w = int(spec["width"][e][l])
            W = params[at: at + w * fan_in].reshape(w, fan_in)
            at += w * fan_in
            b = params[at: at + w]
            at += w
            layers.append((W, b))
            fan_in = w
        c = int(spec["classes"])
        W = params[at: at + c * fan_in].reshape(c, fan_in)
        at += c * fan_in
        b = params[at: at + c]
        at += c
        members.append((layers, (W, b)))
    if at != len(params):
        raise ValueError(f"parameter count {len(params)} != spec's {at}")
    return members


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even), as fp32."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32)


def transform(spec, raw: np.ndarray) -> np.ndarray:
    """z (Q x 19, fp32): x = fp32(raw); t = log1p(max(x, 0)) in fp32 on the
    log_mask dims; z = (t - shift) * scale in fp32."""
    x = np.asarray(raw, np.float64).astype(np.float32)
    mask = int(spec["log_mask"])
    t32 = x.copy()
    for d in range(DIMS):
        if (mask >> d) & 1:
            t32[:, d] = np.log1p(np.maximum(x[:, d], np.float32(0)), dtype=np.float32)
    shift = np.asarray(spec["shift"], np.float32)
    scale = np.asarray(spec["scale"], np.float32)
    return ((t32 - shift).astype(np.float32) * scale).astype(np.float32)


def _ln(x, g, b, eps=1e-5):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def tf_logits(spec, params: np.ndarray, z: np.ndarray) -> np.ndarray:
    """The Transformer ensemble's member logits (Q x E x C) in fp64, parameter
    layout of carma_gpu.h: per member emb W [d x 3], b [d], pos [3 x d]; per
    encoder layer Wq, bq, Wk, bk, Wv, bv, Wo, bo, ln1 g, b, W1 [4 x d], b1,
    W2 [d x 4], b2, ln2 g, b; head H1 [8 x (d + 10)], b, H2 [C x 8], b.
    Tokens: the three layer tuples z[9..17]; auxiliary features z[0..8], z[18];
    post-LN encoder layers (one head, scores / sqrt(d)), mean pooling."""
    E, C = int(spec["members"]), int(spec["classes"])
    p = np.asarray(params, np.float64)
    at = 0

    def take(n, shape=None):
        nonlocal at
        v = p[at: at + n]
        at += n
        return v.reshape(shape) if shape else v

    tok = z[:, 9:18].reshape(-1, 3, 3)
    aux = np.concatenate([z[:, 0:9], z[:, 18:19]], axis=1)
    out = np.zeros((len(z), E, C))
    for e in range(E):
        d, L = int(spec["width"][e][0]), int(spec["depth"][e])
        W, b, pos = take(3 * d, (d, 3)), take(d), take(3 * d, (3, d))
        x = np.maximum(tok @ W.T + b, 0.0) + pos
        for _ in range(L):
            Wq, bq, Wk, bk = take(d * d, (d, d)), take(d), take(d * d, (d, d)), take(d)
            Wv, bv, Wo, bo = take(d * d, (d, d)), take(d), take(d * d, (d, d)), take(d)
            g1, c1 = take(d), take(d)
            W1, b1, W2, b2 = take(4 * d, (4, d)), take(4), take(4 * d, (d, 4)), take(d)
            g2, c2 = take(d), take(d)
            q, k, v = x @ Wq.T + bq, x @ Wk.T + bk, x @ Wv.T + bv
            s = np.einsum("qtd,qud->qtu", q, k) / np.sqrt(d)
            a = np.exp(s - s.max(axis=2, keepdims=True))
            a /= a.sum(axis=2, keepdims=True)
            x = _ln(x + (np.einsum("qtu,qud->qtd", a, v) @ Wo.T + bo), g1, c1)
            x = _ln(x + (np.maximum(x @ W1.T + b1, 0.0) @ W2.T + b2), g2, c2)
        H1, h1, H2, h2 = take(8 * (d + 10), (8, d + 10)), take(8), take(C * 8, (C, 8)), take(C)
        h = np.maximum(np.concatenate([x.mean(axis=1), aux], axis=1) @ H1.T + h1, 0.0)
        out[:, e, :] = h @ H2.T + h2
    if at != len(p):
        raise ValueError(f"parameter count {len(p)} != spec's {at}")
    return out


def forward(spec, params: np.ndarray, raw: np.ndarray):
    """(logits Q x E x C, probs Q x C, bucket Q int32, bytes Q uint64)."""
    z = transform(spec, raw).astype(np.float64)
    if int(spec["arch"]) == 1:  # the Transformer ensemble: fp32 weights
        return _vote(spec, tf_logits(spec, params, z))
    # weights are bf16 values on the device (rounded on install), biases fp32
    members = unpack_params(spec, np.asarray(params, np.float32))
    members = [([(bf16_round(W), b) for W, b in layers], (bf16_round(head[0]), head[1]))
               for layers, head in members]
    E, C = int(spec["members"]), int(spec["classes"])
    logits = np.zeros((len(z), E, C))
    for e, (layers, head) in enumerate(members):
        h = z
        for W, b in layers:
            h = np.maximum(h @ W.astype(np.float64).T + b.astype(np.float64), 0.0)
        logits[:, e, :] = h @ head[0].astype(np.float64).T + head[1].astype(np.float64)
    return _vote(spec, logits)


def _vote(spec, logits):
    """Softmax per member, mean over members, argmax (ties to the larger bin)."""
    C = int(spec["classes"])
    mx = logits.max(axis=2, keepdims=True)
    ex = np.exp(logits - mx)
    probs = (ex / ex.sum(axis=2, keepdims=True)).mean(axis=1)
    # argmax with ties to the larger bin
    bucket = (C - 1 - np.argmax(probs[:, ::-1], axis=1)).astype(np.int32)
    nbytes = (bucket.astype(np.uint64) + np.uint64(1)) * np.uint64(int(spec["bucket_range"]))
    return logits, probs, bucket, nbytes
