"""GPU training backward (train.hpp) against the reference compiled from its
own headers: kan_linear_backward gradients, softmax_cross_entropy, and MLP
SGD-momentum steps.  fp32 on the GPU vs fp64 reference: bar 1e-4 (norm-relative)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2603_17230_b200 import Engine, EvalOptions  # noqa: E402
from paper_2603_17230_b200.engine import softmax_cross_entropy  # noqa: E402
from paper_2603_17230_b200.train import MlpTrainer, TrainConfig  # noqa: E402

TOL = 1e-4


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("G,P,n_in,n_out,M", [(5, 3, 40, 24, 300), (3, 3, 784, 10, 64), (10, 3, 33, 70, 129),
                                              (4, 2, 20, 5, 50), (6, 1, 17, 9, 40)])
def test_linear_backward_matches_reference(ref, G, P, n_in, n_out, M):
    rng = np.random.default_rng(n_in + M)
    W = rng.normal(0, 0.1, (n_in * (G + P), n_out))
    x = rng.uniform(-1.2, 1.2, (M, n_in)).astype(np.float32)
    x[0, :3] = [1.0, -1.0, 0.5]  # the clamp edge and domain ends
    dout = rng.normal(0, 1, (M, n_out)).astype(np.float32)
    desc = {"name": "l", "grid": {"intervals": G, "degree": P}, "input": [n_in],
            "layers": [{"type": "linear", "n_in": n_in, "n_out": n_out}]}
    e = Engine(desc)
    e.set_coeffs(0, W)
    dc, di = e.linear_backward(0, torch.from_numpy(x).cuda(), torch.from_numpy(dout).cuda())
    rc, ri = ref.linear_backward(G, P, x.astype(np.float64), W, dout.astype(np.float64))
    assert _rel(dc.cpu().numpy().astype(np.float64), rc) < TOL
    assert _rel(di.cpu().numpy().astype(np.float64), ri) < TOL
    clamped = (x < -1.0) | (x >= 1.0)
    assert np.all(di.cpu().numpy()[clamped] == 0.0)


def test_softmax_cross_entropy_matches_reference(ref):
    rng = np.random.default_rng(0)
    logits = rng.normal(0, 3, (257, 10)).astype(np.float32)
    labels = rng.integers(0, 10, 257).astype(np.int32)
    loss, d = softmax_cross_entropy(torch.from_numpy(logits).cuda(), torch.from_numpy(labels).cuda())
    rl, rd = ref.softmax_ce(logits.astype(np.float64), labels)
    assert abs(loss - rl) <= 1e-5 * max(1.0, abs(rl))
    assert _rel(d.cpu().numpy().astype(np.float64), rd) < TOL


def test_mlp_sgd_momentum_steps_track_reference(ref):
    """Three minibatch steps of train()'s update rule (train.hpp:338-366) on the
    GPU vs the same steps composed from the reference's functions in fp64."""
    G, P = 5, 3
    dims = [30, 16, 10]
    desc = {"name": "m", "grid": {"intervals": G, "degree": P}, "input": [dims[0]],
            "layers": [{"type": "linear", "n_in": a, "n_out": b} for a, b in zip(dims, dims[1:])]}
    rng = np.random.default_rng(4)
    Ws = [rng.normal(0, 0.2, (a * (G + P), b)) for a, b in zip(dims, dims[1:])]
    cfg = TrainConfig(lr=0.05, momentum=0.9)
    tr = MlpTrainer(desc, Ws, cfg)
    rW = [w.copy() for w in Ws]
    rV = [np.zeros_like(w) for w in Ws]
    for step in range(3):
        x = rng.uniform(-1, 1, (64, dims[0])).astype(np.float32)
        y = rng.integers(0, 10, 64).astype(np.int32)
        loss = tr.step(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
        # reference step in fp64
        acts = [x.astype(np.float64)]
        for w in rW:
            acts.append(ref.linear_forward(G, P, acts[-1], w))
        rloss, d = ref.softmax_ce(acts[-1], y)
        for li in range(len(rW) - 1, -1, -1):
            dc, di = ref.linear_backward(G, P, acts[li], rW[li], d)
            rV[li] = cfg.momentum * rV[li] - cfg.lr * dc
            rW[li] = rW[li] + rV[li]
            d = di
        assert abs(loss - rloss) <= 1e-4 * max(1.0, abs(rloss)), (step, loss, rloss)
        for a, b, w0 in zip(tr.coeffs, rW, Ws):
            assert _rel(a - w0, b - w0) < 1e-3  # the accumulated updates agree
