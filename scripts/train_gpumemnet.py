"""Trains the neural GPUMemNet ensembles and writes
paper_2508_19073_b200/weights/gpumemnet_<family>.npz plus the golden fixture
tests/golden/gpumemnet.npz.

Data: the reference's synthetic estimator datasets (generate_synthetic_dataset,
estimators.cpp:221-264, restated on the host by libcarma_b200), features =
scalar_features (estimators.cpp:317-342), labels = the memory bucket.

Model (paper §4.3, fig. "MLP Ensemble"): 8 members; member m has a random
depth of 1..8 hidden layers whose widths decay exponentially from 8 to 4
neurons; Linear -> BatchNorm -> ReLU per layer; a linear head over the bins;
the ensemble averages the members' softmax outputs. Trained with Adam on
cross-entropy (PyTorch, CPU). Export: batch norm folded into the linear
layers, weights rounded to bf16, biases fp32 — the layout of carma_nn_set_model.

The golden fixture holds raw feature rows and the torch fp64 forward pass of
the exported (folded, rounded) models: the pin for oracle/gpumemnet_oracle.py.

Usage: python scripts/train_gpumemnet.py [--samples 20000] [--epochs 30]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2508_19073_b200 as cb  # noqa: E402
from paper_2508_19073_b200 import gpumemnet as gm  # noqa: E402

CAPACITY = 40 * cb.abi.GiB
MEMBERS = 8


def member_widths(depth: int) -> list:
    if depth == 1:
        return [8]
    return [int(round(8.0 * (0.5 ** (l / (depth - 1))))) for l in range(depth)]


def features(rows: np.ndarray, shift=None, scale=None):
    raw = cb.scalar_features(rows)
    t32 = raw.astype(np.float32)  # the transform of carma_gpu.h, in fp32
    for d in gm.LOG_DIMS:
        t32[:, d] = np.log1p(np.maximum(t32[:, d], np.float32(0)), dtype=np.float32)
    if shift is None:
        shift = t32.mean(axis=0).astype(np.float32)
        sd = t32.std(axis=0).astype(np.float32)
        scale = np.where(sd > 0, 1.0 / np.maximum(sd, 1e-12), 1.0).astype(np.float32)
    z = ((t32 - shift).astype(np.float32) * scale).astype(np.float32)
    return raw, z, shift, scale


class Member(torch.nn.Module):
    def __init__(self, widths, classes):
        super().__init__()
        layers = []
        fan_in = 19
        for w in widths:
            layers += [torch.nn.Linear(fan_in, w), torch.nn.BatchNorm1d(w), torch.nn.ReLU()]
            fan_in = w
        self.body = torch.nn.Sequential(*layers)
        self.head = torch.nn.Linear(fan_in, classes)

    def forward(self, x):
        return self.head(self.body(x))


class TfMember(torch.nn.Module):
    """GPUMemNet Transformer classifier: an MLP input embedding
    of the per-layer tuples (first / middle / last layer: kind, activations,
    params = z[9..17]), learned positional encodings, post-LN encoder layers
    (one head, feed-forward 4), mean pooling, concatenation with the
    structured auxiliary features (z[0..8], z[18]) and an MLP head."""

    def __init__(self, d, layers, classes):
        super().__init__()
        self.d = d
        self.emb = torch.nn.Linear(3, d)
        self.pos = torch.nn.Parameter(torch.randn(3, d) * 0.1)
        self.enc = torch.nn.ModuleList([torch.nn.TransformerEncoderLayer(
            d_model=d, nhead=1, dim_feedforward=4, dropout=0.0, batch_first=True) for _ in range(layers)])
        self.h1 = torch.nn.Linear(d + 10, 8)
        self.h2 = torch.nn.Linear(8, classes)

    def forward(self, z):
        tok = z[:, 9:18].reshape(-1, 3, 3)
        e = torch.relu(self.emb(tok)) + self.pos
        for layer in self.enc:
            e = layer(e)
        aux = torch.cat([z[:, 0:9], z[:, 18:19]], dim=1)
        return self.h2(torch.relu(self.h1(torch.cat([e.mean(dim=1), aux], dim=1))))


def tf_export(m: TfMember) -> list:
    """Flat parameter blocks in the layout of carma_gpu.h (Transformer)."""
    d = m.d
    out = [m.emb.weight, m.emb.bias, m.pos]
    for layer in m.enc:
        w, b = layer.self_attn.in_proj_weight, layer.self_attn.in_proj_bias
        out += [w[:d], b[:d], w[d:2 * d], b[d:2 * d], w[2 * d:], b[2 * d:],
                layer.self_attn.out_proj.weight, layer.self_attn.out_proj.bias,
                layer.norm1.weight, layer.norm1.bias, layer.linear1.weight, layer.linear1.bias,
                layer.linear2.weight, layer.linear2.bias, layer.norm2.weight, layer.norm2.bias]
    out += [m.h1.weight, m.h1.bias, m.h2.weight, m.h2.bias]
    return [t.detach().float().numpy().ravel() for t in out]


def fold(member: Member) -> list:
    """[(W, b)] per hidden layer with batch norm folded, then the head."""
    out = []
    mods = list(member.body)
    for i in range(0, len(mods), 3):
        lin, bn = mods[i], mods[i + 1]
        s = (bn.weight / torch.sqrt(bn.running_var + bn.eps)).double()
        W = lin.weight.double() * s[:, None]
        b = (lin.bias.double() - bn.running_mean.double()) * s + bn.bias.double()
        out.append((W, b))
    out.append((member.head.weight.double(), member.head.bias.double()))
    return out


def bf16(x: torch.Tensor) -> torch.Tensor:
    return x.float().to(torch.bfloat16).float()


def export_params(folded_members) -> np.ndarray:
    flat = []
    for layers in folded_members:
        for W, b in layers:
            flat.append(bf16(W).numpy().ravel())
            flat.append(b.float().numpy().ravel())
    return np.concatenate(flat).astype(np.float32)


def torch_forward(folded_members, z: np.ndarray) -> np.ndarray:
    """fp64 forward of the exported model (rounded weights, fp32 biases)."""
    x = torch.from_numpy(z.astype(np.float64))
    outs = []
    for layers in folded_members:
        h = x
        for i, (W, b) in enumerate(layers):
            h = h @ bf16(W).double().T + b.float().double()
            if i + 1 < len(layers):
                h = torch.relu(h)
        outs.append(h)
    return torch.stack(outs, dim=1).numpy()


def train_members(build, n_members, xt, yt, epochs):
    members = []
    n = len(xt)
    for e in range(n_members):
        m = build(e)
        opt = torch.optim.Adam(m.parameters(), lr=1e-2)
        sched = torch.optim.lr_scheduler.CosineAnnealingLR(opt, epochs)
        m.train()
        for _ in range(epochs):
            order = torch.randperm(n)
            for i in range(0, n, 256):
                idx = order[i: i + 256]
                if len(idx) < 2:
                    continue
                opt.zero_grad()
                loss = torch.nn.functional.cross_entropy(m(xt[idx]), yt[idx])
                loss.backward()
                opt.step()
            sched.step()
        m.eval()
        members.append(m)
    return members


def train_family_tf(family: int, samples: int, epochs: int, seed: int):
    """The Transformer ensemble: 8 members, d in {4, 6}, 2-3 encoder layers
    (PAPER.md:440), weights exported unrounded (fp32; the Transformer kernel
    runs on the CUDA cores)."""
    torch.manual_seed(seed)
    rng = np.random.default_rng(seed)
    ds = cb.generate_synthetic_dataset(family, samples, 1000 + family)
    br = ds.bucket_range
    classes = CAPACITY // br + 1
    raw, z, shift, scale = features(ds.rows)
    y = np.minimum(ds.bucket, classes - 1).astype(np.int64)
    n_train = int(0.8 * samples)
    perm = rng.permutation(samples)
    tr, ho = perm[:n_train], perm[n_train:]
    dims = [int(v) for v in rng.choice([4, 6], size=MEMBERS)]
    layers = [int(v) for v in rng.integers(2, 4, size=MEMBERS)]
    members = train_members(lambda e: TfMember(dims[e], layers[e], classes), MEMBERS,
                            torch.from_numpy(z[tr]), torch.from_numpy(y[tr]), epochs)
    with torch.no_grad():
        logits = torch.stack([m(torch.from_numpy(z[ho])) for m in members], dim=1).double().numpy()
    probs = torch.softmax(torch.from_numpy(logits), dim=2).mean(dim=1).numpy()
    pred = classes - 1 - np.argmax(probs[:, ::-1], axis=1)
    acc = float((pred == y[ho]).mean())
    params = np.concatenate([np.concatenate(tf_export(m)) for m in members]).astype(np.float32)
    model = gm.NnModel(family, br, classes, layers, [[d] for d in dims], shift, scale, params, gm.LOG_MASK, acc,
                       arch=gm.ARCH_TRANSFORMER)
    return model, members


def train_family(family: int, samples: int, epochs: int, seed: int):
    torch.manual_seed(seed)
    rng = np.random.default_rng(seed)
    ds = cb.generate_synthetic_dataset(family, samples, 1000 + family)
    br = ds.bucket_range
    classes = CAPACITY // br + 1
    raw, z, shift, scale = features(ds.rows)
    y = np.minimum(ds.bucket, classes - 1).astype(np.int64)
    n_train = int(0.8 * samples)
    perm = rng.permutation(samples)
    tr, ho = perm[:n_train], perm[n_train:]
    xt = torch.from_numpy(z[tr])
    yt = torch.from_numpy(y[tr])
    depths = [int(d) for d in rng.integers(1, 9, size=MEMBERS)]
    members = []
    for e, d in enumerate(depths):
        m = Member(member_widths(d), classes)
        opt = torch.optim.Adam(m.parameters(), lr=1e-2)
        sched = torch.optim.lr_scheduler.CosineAnnealingLR(opt, epochs)
        m.train()
        for _ in range(epochs):
            order = torch.randperm(n_train)
            for i in range(0, n_train, 256):
                idx = order[i: i + 256]
                if len(idx) < 2:
                    continue
                opt.zero_grad()
                loss = torch.nn.functional.cross_entropy(m(xt[idx]), yt[idx])
                loss.backward()
                opt.step()
            sched.step()
        m.eval()
        members.append(m)
    with torch.no_grad():
        folded = [fold(m) for m in members]
        logits = torch_forward(folded, z[ho])
    probs = torch.softmax(torch.from_numpy(logits), dim=2).mean(dim=1).numpy()
    pred = classes - 1 - np.argmax(probs[:, ::-1], axis=1)
    acc = float((pred == y[ho]).mean())
    params = export_params(folded)
    model = gm.NnModel(family, br, classes, depths, [member_widths(d) for d in depths], shift, scale, params,
                       gm.LOG_MASK, acc)
    return model, folded


def main_tf(args) -> None:
    golden = {}
    for family, name in gm.FAMILY_NAMES.items():
        t0 = time.time()
        model, members = train_family_tf(family, args.samples, args.epochs, seed=17 + family)
        model.save(os.path.join(gm.WEIGHTS_DIR, f"gpumemnet_tf_{name}.npz"))
        ds = cb.generate_synthetic_dataset(family, 256, 4242 + family)
        raw, z, _, _ = features(ds.rows, model.shift, model.scale)
        with torch.no_grad():
            zz = torch.from_numpy(z.astype(np.float64))
            logits = torch.stack([m.double()(zz) for m in members], dim=1).numpy()
        golden[f"{name}_rows"] = ds.rows.view(np.uint8).reshape(len(ds.rows), -1)
        golden[f"{name}_raw"] = raw
        golden[f"{name}_logits"] = logits.astype(np.float32)
        golden[f"{name}_labels"] = ds.bucket
        print(f"transformer {name}: classes {model.classes}, layers {model.depth}, d {[w[0] for w in model.width]}, "
              f"holdout accuracy {model.holdout_accuracy:.4f}, {time.time() - t0:.1f} s")
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "gpumemnet_tf.npz"), **golden)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=20000)
    ap.add_argument("--epochs", type=int, default=30)
    ap.add_argument("--arch", choices=("mlp", "transformer"), default="mlp")
    args = ap.parse_args()
    os.makedirs(gm.WEIGHTS_DIR, exist_ok=True)
    if args.arch == "transformer":
        main_tf(args)
        return
    golden = {}
    for family, name in gm.FAMILY_NAMES.items():
        t0 = time.time()
        model, folded = train_family(family, args.samples, args.epochs, seed=7 + family)
        model.save(os.path.join(gm.WEIGHTS_DIR, f"gpumemnet_{name}.npz"))
        # golden: 256 fresh rows of the family (a different dataset seed)
        ds = cb.generate_synthetic_dataset(family, 256, 4242 + family)
        raw, z, _, _ = features(ds.rows, model.shift, model.scale)
        with torch.no_grad():
            logits = torch_forward(folded, z)
        golden[f"{name}_rows"] = ds.rows.view(np.uint8).reshape(len(ds.rows), -1)
        golden[f"{name}_raw"] = raw
        golden[f"{name}_logits"] = logits.astype(np.float32)
        golden[f"{name}_labels"] = ds.bucket
        print(f"{name}: classes {model.classes}, depths {model.depth}, holdout accuracy "
              f"{model.holdout_accuracy:.4f}, {time.time() - t0:.1f} s")
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "gpumemnet.npz"), **golden)


if __name__ == "__main__":
    main()
