"""GPU tests of the integration around the hot path: the training step (fused
RMSNorm + LCE, then Layer-Adam on dW) against an fp64 oracle loop, autograd with per-row upstream
gradients, and CUDA-graph capture of the fused call."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import GRAD_TOL, assert_loss_close, bf16_to_np64, oracle_inputs, rel_max_err, to_dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_16428_b200 as m
    return m


def test_train_loop_vs_oracle_loop(slf):
    """K = 3 steps of LMHeadTrainer on the tiny config (a fresh seeded batch per step) against the
    oracle loop: loss_k, dW_k = oracle.rmsnorm_lce(x_k, g, bf16(p)), p = oracle.adam_step(p, dW_k).

    Tolerance, derived from the north-star gradient bound: the Adam update
    u = lr m^/(sqrt(v^) + eps) changes by at most lr/eps per unit change of m^ and of sqrt(v^), and
    both move by at most the gradient error d_k = GRAD_TOL * max|dW_k| (max norm), so after K steps
    |p_gpu - p_oracle| <= sum_k 2 lr max_{j<=k} d_j / eps.  eps = 1e-2 (above the largest |dW|
    here, ~4e-3) keeps that bound below the parameters' movement; as eps -> 0 the first Adam step
    becomes lr * sign(g) and entries whose |g| is below the bf16 gradient error can flip — the bound
    grows as 1/eps, i.e. the comparison, not the code, becomes ill-conditioned.  The worst-case
    bound is loose (about half the movement here); the error is also held to GRAD_TOL of the
    movement (observed on the B200: 1.8e-5 against 1.9e-3, about 1 %)."""
    from paper_2603_16428_b200.train import LMHeadTrainer
    K, lr, eps = 3, 1e-3, 1e-2
    base = synth.make_config("tiny", seed=50, alpha=4.0, dist="zipf")
    H = base.H
    g_np = synth.f32_to_bf16_bits((1 + 0.2 * np.random.default_rng(7).standard_normal(H)).astype(np.float32))
    g = torch.from_numpy(g_np.view(np.int16)).view(torch.bfloat16).cuda()
    _, W, _ = to_dev(base, torch)
    W0 = W.clone()
    tr = LMHeadTrainer(W, g, lr=lr, eps=eps)
    batches = [synth.make_config("tiny", seed=60 + k, alpha=4.0, dist="zipf") for k in range(K)]
    losses = []
    for b in batches:
        x, _, t = to_dev(b, torch)
        loss, dx, dg = tr.step(x, t)
        losses.append(float(loss))
    p_gpu, m_gpu, v_gpu, steps = tr.master()
    torch.cuda.synchronize()
    assert steps == K
    # the device copy of W is the RNE bf16 rounding of the host master
    assert np.array_equal(W.view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1),
                          oracle.bf16_rne(p_gpu.numpy().astype(np.float64)))
    # oracle loop (fp64)
    p = synth.bf16_bits_to_f64(base.W).reshape(-1)
    p0 = p.copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    gw = synth.bf16_bits_to_f64(g_np)
    bound, dmax = 0.0, 0.0
    for k, b in enumerate(batches):
        W_used = synth.bf16_bits_to_f64(oracle.bf16_rne(p)).reshape(base.V, H)
        xo, _, to = oracle_inputs(b)
        loss_k, _, _, dW = oracle.rmsnorm_lce(xo, gw, W_used, to, eps=1e-5, reduction="mean")
        assert_loss_close(losses[k], loss_k, "mean")
        p, m, v = oracle.adam_step(p, m, v, dW.reshape(-1), k + 1, lr, eps=eps)
        dmax = max(dmax, GRAD_TOL * np.max(np.abs(dW)))
        bound += 2 * lr * dmax / eps
    moved = np.max(np.abs(p - p0))
    err = np.max(np.abs(p_gpu.numpy().astype(np.float64) - p))
    print(f"train loop: max |p_gpu - p_oracle| = {err:.3e} (bound {bound:.3e}), max movement {moved:.3e}, "
          f"losses {losses}")
    assert err <= bound
    assert err <= GRAD_TOL * moved  # and, observed, within the gradient tolerance of the movement
    assert not torch.equal(W, W0)
    tr.close()


@pytest.mark.parametrize("red", ["none", "mean"])
def test_lce_function_upstream_grad_on_device(slf, red):
    """LCEFunction (schedule-R split) with an upstream gradient that is a device tensor — per row for
    reduction='none' — folded into the RowStat coefficients on the device: gradients of
    sum_i w_i * loss_i against the oracle rows with coef_i = w_i * valid_i."""
    inp = synth.make_inputs(500, 256, 3000, seed=29, alpha=3.0, dist="zipf")
    X, W, t = to_dev(inp, torch)
    Xr = X.clone().requires_grad_(True)
    Wr = W.clone().requires_grad_(True)
    L = slf.LCEFunction.apply(Xr, Wr, t, -100, red)
    rng = np.random.default_rng(3)
    w = rng.uniform(-1.5, 2.0, size=500) if red == "none" else np.array([0.75])
    wt = torch.from_numpy(w.astype(np.float32)).cuda()
    (L * (wt if red == "none" else wt[0])).sum().backward()
    torch.cuda.synchronize()
    Xo, Wo, to = oracle_inputs(inp)
    valid, nv, coef = oracle.coef_for(to, -100, red, 1.0)
    coef = coef * (w if red == "none" else w[0])
    l, _, dXo, G = oracle.rows(Xo, Wo, to, coef)
    dWo = G.T @ Xo
    assert rel_max_err(bf16_to_np64(Xr.grad), dXo) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(Wr.grad), dWo) <= GRAD_TOL
    if red == "none":
        assert_loss_close(L.detach().cpu().numpy(), l, "none")


def test_fused_call_cuda_graph_capture(slf):
    """The fused call captured in a CUDA graph (tile tables uploaded from persistent pinned copies):
    replaying it on new contents of the static input buffers gives bit-identical results to eager
    calls on those inputs."""
    a = synth.make_inputs(1100, 256, 3000, seed=31, alpha=4.0, dist="zipf")
    b = synth.make_inputs(1100, 256, 3000, seed=32, alpha=1.0, dist="uniform")
    Xa, W, ta = to_dev(a, torch)
    Xb, _, tb = to_dev(b, torch)
    budget = 2 << 20
    ws = slf.alloc_workspace(1100, 256, 3000, Xa.device, "S", budget)
    X, t = Xa.clone(), ta.clone()
    out = (torch.empty(1, device="cuda"), torch.empty_like(X), torch.empty_like(W))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        slf.lce_fwd_bwd(X, W, t, out=out, workspace=ws, budget_bytes=budget, schedule="S")
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        slf.lce_fwd_bwd(X, W, t, out=out, workspace=ws, budget_bytes=budget, schedule="S")
    for Xn, tn in ((Xb, tb), (Xa, ta)):
        X.copy_(Xn)
        t.copy_(tn)
        graph.replay()
        torch.cuda.synchronize()
        ref = slf.lce_fwd_bwd(Xn, W, tn, budget_bytes=budget, schedule="S")
        torch.cuda.synchronize()
        assert torch.equal(out[0].view(-1), ref[0].view(-1))
        assert torch.equal(out[1], ref[1]) and torch.equal(out[2], ref[2])
