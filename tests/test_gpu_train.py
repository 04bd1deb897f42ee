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


CNN = {"name": "cnn", "grid": {"intervals": 3, "degree": 3}, "input": [2, 11, 11],
       "layers": [{"type": "conv", "c_in": 2, "c_out": 4, "kernel": 3, "stride": 1, "padding": 1},
                  {"type": "maxpool", "window": 2},
                  {"type": "conv", "c_in": 4, "c_out": 5, "kernel": 3, "stride": 2, "padding": 1},
                  {"type": "flatten"},
                  {"type": "linear", "n_in": 45, "n_out": 10}]}


def _cnn_ws(seed):
    rng = np.random.default_rng(seed)
    nb = 6
    return [rng.normal(0, 0.3, (2 * 9 * nb, 4)), rng.normal(0, 0.3, (4 * 9 * nb, 5)),
            rng.normal(0, 0.3, (45 * nb, 10))]


@pytest.mark.parametrize("desc_ws", ["mlp", "cnn"])
def test_training_tracks_reference_train(ref, desc_ws):
    """Two full-batch epochs of the reference's own train() (train.hpp:247-462)
    vs the GPU Trainer: updated coefficients and loss."""
    import json
    from paper_2603_17230_b200.train import Trainer
    if desc_ws == "mlp":
        desc = {"name": "m", "grid": {"intervals": 5, "degree": 3}, "input": [30],
                "layers": [{"type": "linear", "n_in": 30, "n_out": 16},
                           {"type": "linear", "n_in": 16, "n_out": 10}]}
        rng = np.random.default_rng(8)
        Ws = [rng.normal(0, 0.2, (30 * 8, 16)), rng.normal(0, 0.2, (16 * 8, 10))]
    else:
        desc, Ws = CNN, _cnn_ws(9)
    D = int(np.prod(desc["input"]))
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, (48, D)).astype(np.float32)
    y = rng.integers(0, 10, 48).astype(np.int32)
    cfg = TrainConfig(lr=0.05, momentum=0.9)
    tr = Trainer(desc, Ws, cfg)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for _ in range(2):
        loss = tr.step(xd, yd)
    rW, rloss = ref.train(json.dumps(desc), Ws, x.astype(np.float64), y, cfg.lr, cfg.momentum, 2, 48)
    assert abs(loss - rloss) <= 1e-4 * max(1.0, abs(rloss)), (loss, rloss)
    for a, b, w0 in zip(tr.coeffs, rW, Ws):
        assert _rel(a - w0, b - w0) < 1e-3


def test_conv_backward_matches_reference_composition(ref):
    """kan_engine_conv_backward vs the reference's conv step: im2col patches,
    kan_linear_backward on the patch rows, col2im_add (train.hpp:367-399)."""
    G, P = 3, 3
    rng = np.random.default_rng(3)
    c_in, c_out, H, W = 3, 6, 7, 7
    desc = {"name": "c", "grid": {"intervals": G, "degree": P}, "input": [c_in, H, W],
            "layers": [{"type": "conv", "c_in": c_in, "c_out": c_out, "kernel": 3, "stride": 2, "padding": 1}]}
    Wt = rng.normal(0, 0.3, (c_in * 9 * (G + P), c_out))
    e = Engine(desc)
    e.set_coeffs(0, Wt)
    M = 5
    x = rng.uniform(-1.1, 1.1, (M, c_in, H, W)).astype(np.float32)
    Ho = (H + 2 - 3) // 2 + 1
    dout = rng.normal(0, 1, (M, c_out, Ho, Ho)).astype(np.float32)
    dc, di = e.conv_backward(0, torch.from_numpy(x).cuda(), torch.from_numpy(dout).cuda())
    rdc = np.zeros_like(Wt)
    rdi = np.zeros(x.shape)
    for m in range(M):
        patches = ref.im2col(x[m].astype(np.float64), 3, 2, 1)
        drows = dout[m].reshape(c_out, -1).T.astype(np.float64)
        gc, gi = ref.linear_backward(G, P, patches, Wt, drows)
        rdc += gc
        for oy in range(Ho):
            for ox in range(Ho):
                row = gi[oy * Ho + ox]
                col = 0
                for c in range(c_in):
                    for ky in range(3):
                        for kx in range(3):
                            iy, ix = oy * 2 + ky - 1, ox * 2 + kx - 1
                            if 0 <= iy < H and 0 <= ix < W:
                                rdi[m, c, iy, ix] += row[col]
                            col += 1
    assert _rel(dc.cpu().numpy().astype(np.float64), rdc) < TOL
    assert _rel(di.cpu().numpy().astype(np.float64), rdi) < TOL


def test_sgd_step_on_device_is_the_reference_update():
    """kan_engine_sgd_step: v = momentum*v - lr*g; w += v in fp64 on the device
    master copy (train.hpp:361-366) -- bit-identical to the same fp64 arithmetic
    on the host for the fp32 gradients it is given; the fp32 forward and backward
    read the updated weights; set_coeffs resets the momentum."""
    G, P, n_in, n_out, M = 5, 3, 37, 12, 65
    rng = np.random.default_rng(5)
    W = rng.normal(0, 0.1, (n_in * (G + P), n_out))
    desc = {"name": "l", "grid": {"intervals": G, "degree": P}, "input": [n_in],
            "layers": [{"type": "linear", "n_in": n_in, "n_out": n_out}]}
    e = Engine(desc)
    e.set_coeffs(0, W)
    e.configure(EvalOptions(mode="fp32"))
    x = torch.from_numpy(rng.uniform(-1, 1, (M, n_in)).astype(np.float32)).cuda()
    w, v = W.copy(), np.zeros_like(W)
    lr, mom = 0.05, 0.9
    for step in range(3):
        dout = torch.from_numpy(rng.normal(0, 1, (M, n_out)).astype(np.float32)).cuda()
        dc, _ = e.linear_backward(0, x, dout)
        e.sgd_step(0, dc, lr, mom)
        v = mom * v - lr * dc.cpu().numpy().astype(np.float64)
        w = w + v
        np.testing.assert_array_equal(e.get_coeffs(0), w)
    # the forward reads the updated weights: equal to a fresh engine on them
    y = e.model_forward(x).cpu().numpy()
    f = Engine(desc)
    f.set_coeffs(0, w)
    f.configure(EvalOptions(mode="fp32"))
    np.testing.assert_array_equal(y, f.model_forward(x).cpu().numpy())
    # and so does the backward (its fp32 copy was refreshed in the same launch)
    dout = torch.from_numpy(rng.normal(0, 1, (M, n_out)).astype(np.float32)).cuda()
    _, di = e.linear_backward(0, x, dout)
    _, di_f = f.linear_backward(0, x, dout)
    np.testing.assert_array_equal(di.cpu().numpy(), di_f.cpu().numpy())
    # reconfiguring keeps the trained coefficients; set_coeffs restarts the momentum
    e.configure(EvalOptions(mode="fp32"))
    np.testing.assert_array_equal(e.get_coeffs(0), w)
    e.set_coeffs(0, W)
    e.configure(EvalOptions(mode="fp32"))
    dc, _ = e.linear_backward(0, x, dout)
    e.sgd_step(0, dc, lr, mom)
    np.testing.assert_array_equal(e.get_coeffs(0), W - lr * dc.cpu().numpy().astype(np.float64))
