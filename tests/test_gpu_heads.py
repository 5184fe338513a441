"""GPU parity on every BASELINE.json head (``-m gpu``, slow): the CUDA path through the C ABI against
the fp64 oracle on the same seeded inputs.  Tolerances (BASELINE.json north_star): loss relative
1e-3, dX and dW max|err| <= 2e-2 * max|ref|, ignore masking bit-exact.

* reduced N at the head's full H and V, every element, with a budget that forces several row chunks
  (so the multi-chunk bf16 dW reduce-add is compared with the oracle, not only a single chunk);
* full N, H, V in the launch configuration bench.py times (default plan, 5 % budget): dW rows (the
  most-hit Zipf rows and random rows) and dX rows, from the oracle's lse over ALL rows (materialised
  logits row block by row block);
* gradient accumulation (SLF_FLAG_ACCUMULATE_DW) against the oracle's dW_a + dW_b.
"""
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


def _plan(slf, N, H, V, budget, sched):
    desc = slf.plan_describe(N, H, V, budget_bytes=budget, schedule=sched)
    return desc, dict(x.split("=", 1) for x in desc.split() if "=" in x)


def _check_full(slf, inp, budget, sched, reduction="mean", ref=None):
    X, W, t = to_dev(inp, torch)
    loss, dX, dW = slf.lce_fwd_bwd(X, W, t, reduction=reduction, budget_bytes=budget, schedule=sched)
    torch.cuda.synchronize()
    if ref is None:
        ref = oracle.lce(*oracle_inputs(inp), reduction=reduction)
    assert_loss_close(loss.cpu().numpy(), ref["loss"], reduction)
    ex, ew = rel_max_err(bf16_to_np64(dX), ref["dX"]), rel_max_err(bf16_to_np64(dW), ref["dW"])
    assert ex <= GRAD_TOL, f"dX rel max err {ex}"
    assert ew <= GRAD_TOL, f"dW rel max err {ew}"
    assert np.all(dX.view(torch.int16).cpu().numpy()[inp.t == -100] == 0)
    return ex, ew, ref


# ---- reduced N, full H and V, several chunks -------------------------------------------------------
_REF = {}


@pytest.mark.slow
@pytest.mark.parametrize("sched", ["S", "R"])
def test_llama70b_reduced_n_multichunk(slf, sched):
    """Llama-3.1-70B head (H=8192, V=128256) at N=1024, every element, budget 70 MB: schedule S runs
    4 row chunks of 256 (dW accumulated by 3 bf16 reduce-adds), schedule R several row blocks /
    vocab chunks."""
    N, H, V = 1024, 8192, 128256
    budget = 70 << 20
    desc, kv = _plan(slf, N, H, V, budget, sched)
    if sched == "S":
        assert int(kv["n_chunks"]) >= 3, desc
    else:
        assert int(kv["n_row_blocks"]) * int(kv["n_vocab_chunks"]) >= 3, desc
    inp = synth.make_config("llama70b", seed=41, alpha=4.0, dist="zipf", N=N)
    ex, ew, _REF["llama70b"] = _check_full(slf, inp, budget, sched, ref=_REF.get("llama70b"))
    print(f"llama70b N={N} {sched} [{desc}]: dX err {ex:.2e} dW err {ew:.2e}")


@pytest.mark.slow
@pytest.mark.parametrize("sched", ["S", "R"])
def test_mistral_reduced_n_multichunk(slf, sched):
    """Mistral-Large head (H=12288, V=32768) at N=2048 with a 20 MB budget: several row chunks (S:
    extended chunks of 512 rows, bf16 reduce-add dW across them) against every oracle element."""
    N, H, V = 2048, 12288, 32768
    budget = 20 << 20
    desc, kv = _plan(slf, N, H, V, budget, sched)
    if sched == "S":
        assert int(kv["n_chunks"]) >= 3, desc
    inp = synth.make_config("mistral123b", seed=42, alpha=4.0, dist="zipf", N=N)
    ex, ew, _REF["mistral"] = _check_full(slf, inp, budget, sched, ref=_REF.get("mistral"))
    print(f"mistral123b N={N} {sched} [{desc}]: dX err {ex:.2e} dW err {ew:.2e}")


@pytest.mark.slow
def test_qwen_reduced_n_multichunk(slf):
    """Qwen2.5-7B head (H=3584, V=152064) at N=2048, 100 MB budget: S with >= 4 row chunks."""
    N, H, V = 2048, 3584, 152064
    budget = 100 << 20
    desc, kv = _plan(slf, N, H, V, budget, "S")
    assert int(kv["n_chunks"]) >= 4, desc
    inp = synth.make_config("qwen7b", seed=43, alpha=4.0, dist="zipf", N=N)
    ex, ew, _ = _check_full(slf, inp, budget, "S", reduction="sum")
    print(f"qwen7b N={N} S [{desc}]: dX err {ex:.2e} dW err {ew:.2e}")


# ---- gradient accumulation against the oracle ------------------------------------------------------
@pytest.mark.parametrize("sched", ["R", "S"])
def test_accumulate_dw_vs_oracle(slf, sched):
    """dW of micro-batch a, then micro-batch b accumulated into it (accumulate_dw=True), against the
    oracle's dW_a + dW_b; b's loss and dX against the oracle on b alone."""
    a = synth.make_inputs(600, 256, 3000, seed=17, alpha=3.0, dist="zipf")
    b = synth.make_inputs(700, 256, 3000, seed=18, alpha=3.0)
    b.W = a.W
    Xa, W, ta = to_dev(a, torch)
    Xb, _, tb = to_dev(b, torch)
    _, _, acc = slf.lce_fwd_bwd(Xa, W, ta, reduction="sum", scale=0.5, schedule=sched, budget_bytes=2 << 20)
    loss = torch.empty(1, dtype=torch.float32, device="cuda")
    dX = torch.empty_like(Xb)
    slf.lce_fwd_bwd(Xb, W, tb, reduction="sum", scale=0.5, schedule=sched, budget_bytes=2 << 20,
                    out=(loss, dX, acc), accumulate_dw=True)
    torch.cuda.synchronize()
    ra = oracle.lce(*oracle_inputs(a), reduction="sum", scale=0.5)
    rb = oracle.lce(*oracle_inputs(b), reduction="sum", scale=0.5)
    assert_loss_close(float(loss), rb["loss"], "sum")
    assert rel_max_err(bf16_to_np64(dX), rb["dX"]) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(acc), ra["dW"] + rb["dW"]) <= GRAD_TOL


# ---- full size, the bench's launch configuration: dW rows and dX rows ------------------------------
def _oracle_lse_all_rows(inp, Wo, tt, block=1024):
    """lse_i and z_{i,t_i} for every row of the full problem (c1-c2: materialised logits, row blocks
    of whole rows)."""
    lse = np.empty(inp.N)
    zt = np.empty(inp.N)
    for s in range(0, inp.N, block):
        Xb = synth.bf16_bits_to_f64(inp.X[s:s + block])
        Z = Xb @ Wo.T
        m = Z.max(axis=1)
        lse[s:s + block] = m + np.log(np.exp(Z - m[:, None]).sum(axis=1))
        zt[s:s + block] = Z[np.arange(Z.shape[0]), tt[s:s + block]]
    return lse, zt


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["llama8b", "qwen7b", "mistral123b", "llama70b"])
def test_full_size_dw_and_dx_rows(slf, cfg):
    """Every BASELINE head at full N, H, V with the default plan (as bench.py runs it), Zipf targets
    with trained-like logits (alpha 4): 12 dW rows (the 6 most-hit vocabulary rows and 6 random ones)
    and 16 dX rows (incl. 2 ignored, which must be exactly +0.0) against the fp64 oracle; loss (mean)
    against the oracle's lse over all rows."""
    inp = synth.make_config(cfg, seed=2, alpha=4.0, dist="zipf")
    X, W, t = to_dev(inp, torch)
    loss, dX, dW = slf.lce_fwd_bwd(X, W, t, reduction="mean")
    torch.cuda.synchronize()
    valid, nv, coef = oracle.coef_for(inp.t, -100, "mean", 1.0)
    rng = np.random.default_rng(4)
    hot = np.argsort(-np.bincount(inp.t[valid], minlength=inp.V), kind="stable")[:6]
    vrows = np.unique(np.concatenate([hot, rng.choice(inp.V, 6, replace=False)]))
    xrows = np.sort(np.concatenate([rng.choice(np.nonzero(valid)[0], 14, replace=False),
                                    np.nonzero(~valid)[0][:2]]))
    got_w = bf16_to_np64(dW[torch.from_numpy(vrows).cuda()])
    got_x = bf16_to_np64(dX[torch.from_numpy(xrows).cuda()])
    got_loss = float(loss)
    del X, W, t, dX, dW
    torch.cuda.empty_cache()
    Wo = synth.bf16_bits_to_f64(inp.W)
    tt = np.where(valid, inp.t, 0).astype(np.int64)
    lse, zt = _oracle_lse_all_rows(inp, Wo, tt)
    ref_loss = float(np.where(valid, lse - zt, 0.0).sum() / nv)
    assert_loss_close(got_loss, ref_loss, "mean")
    # dW rows vrows: sum_i coef_i (p_iv - [t_i = v]) x_i  (c3), all N tokens, in row blocks
    ref_w = np.zeros((len(vrows), inp.H))
    for s in range(0, inp.N, 4096):
        Xb = synth.bf16_bits_to_f64(inp.X[s:s + 4096])
        P = np.exp(Xb @ Wo[vrows].T - lse[s:s + 4096, None])
        onehot = (inp.t[s:s + 4096, None] == vrows[None, :]).astype(np.float64)
        ref_w += (coef[s:s + 4096, None] * (P - onehot)).T @ Xb
    assert rel_max_err(got_w, ref_w) <= GRAD_TOL, cfg
    # dX rows: the oracle's own row routine (full V columns of those rows)
    _, _, ref_x, _ = oracle.rows(synth.bf16_bits_to_f64(inp.X[xrows]), Wo, inp.t[xrows].astype(np.int64),
                                 coef[xrows])
    assert rel_max_err(got_x, ref_x) <= GRAD_TOL, cfg
    assert np.all(got_x[~valid[xrows]] == 0) and not np.signbit(got_x[~valid[xrows]]).any()
    print(f"{cfg}: dW rows err {rel_max_err(got_w, ref_w):.2e}, dX rows err {rel_max_err(got_x, ref_x):.2e}, "
          f"hits of hottest row {np.bincount(inp.t[valid]).max()}")
