"""GPU parity tests (``-m gpu``): the CUDA path through the C ABI against the fp64 oracle on the
same seeded inputs.  Tolerances (BASELINE.json north_star): loss relative 1e-3, dX and dW
max|err| <= 2e-2 * max|ref|; integer masking bit-exact.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from gpu_util import (GRAD_TOL, assert_loss_close, bf16_to_np64, oracle_inputs, rel_max_err, to_dev)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def slf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_16428_b200 as m
    return m


SCHEDS = ["R", "S"]


def run_gpu(slf, inp, reduction="mean", scale=1.0, budget=0, ignore_index=-100, schedule="auto"):
    X, W, t = to_dev(inp, torch)
    loss, dX, dW = slf.lce_fwd_bwd(X, W, t, ignore_index=ignore_index, reduction=reduction, scale=scale,
                                   budget_bytes=budget, schedule=schedule)
    torch.cuda.synchronize()
    return loss, dX, dW


def check_against_oracle(slf, inp, reduction="mean", scale=1.0, budget=0, ignore_index=-100, schedule="auto"):
    loss, dX, dW = run_gpu(slf, inp, reduction, scale, budget, ignore_index, schedule)
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, ignore_index=ignore_index, reduction=reduction, scale=scale)
    assert_loss_close(loss.detach().cpu().numpy(), ref["loss"], reduction)
    gx = bf16_to_np64(dX)
    gw = bf16_to_np64(dW)
    ex, ew = rel_max_err(gx, ref["dX"]), rel_max_err(gw, ref["dW"])
    assert ex <= GRAD_TOL, f"dX rel max err {ex}"
    assert ew <= GRAD_TOL, f"dW rel max err {ew}"
    ign = inp.t == ignore_index
    if ign.any():  # ignored rows are exactly +0.0 (bf16 bits 0x0000)
        bits = dX.view(torch.int16).cpu().numpy()[ign]
        assert np.all(bits == 0)
    return ex, ew


# ---- the GEMM core alone -------------------------------------------------------------------------
@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", [(128, 256, 64), (384, 512, 320), (200, 264, 136), (1024, 768, 2048)])
def test_gemm_core(slf, a_mn, b_mn, shape):
    M, N, K = shape
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(K, N, generator=g).to(torch.bfloat16)
    ref = (A.double() @ B.double()).numpy()
    Ad = (A.t().contiguous() if a_mn else A).cuda()           # a_mn: stored [K, M]
    Bd = (B.contiguous() if b_mn else B.t().contiguous()).cuda()  # b_mn: stored [K, N]; else [N, K]
    D = slf.debug_gemm(Ad, Bd, a_mn, b_mn, M, N, K)
    torch.cuda.synchronize()
    err = rel_max_err(D.cpu().numpy(), ref)
    assert err < 1e-5, err


# ---- full path vs oracle -------------------------------------------------------------------------
@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("reduction", ["mean", "sum", "none"])
@pytest.mark.parametrize("alpha,dist", [(1.0, "uniform"), (4.0, "zipf"), (4.0, "uniform")])
def test_tiny_parity(slf, reduction, alpha, dist, sched):
    inp = synth.make_config("tiny", seed=11, alpha=alpha, dist=dist)
    check_against_oracle(slf, inp, reduction=reduction, scale=1.0 if reduction != "sum" else 0.25, schedule=sched)


def test_multichunk_ragged_parity_r(slf):
    """Schedule R: several row blocks and vocab chunks, ragged tails in every GEMM dimension."""
    inp = synth.make_inputs(1000, 200, 5000, seed=5, alpha=4.0, dist="zipf")
    budget = 5 << 18  # 1.25 MiB forces nR > 1 and nC > 1
    desc = slf.plan_describe(1000, 200, 5000, budget_bytes=budget, schedule="R")
    kv = dict(x.split("=") for x in desc.split())
    assert int(kv["n_row_blocks"]) > 1 and int(kv["n_vocab_chunks"]) > 1, desc
    check_against_oracle(slf, inp, reduction="mean", budget=budget, schedule="R")
    check_against_oracle(slf, inp, reduction="none", budget=budget, schedule="R")


@pytest.mark.parametrize("reduction", ["mean", "none"])
def test_multichunk_ragged_parity_s(slf, reduction):
    """Schedule S: several row chunks (ragged last chunk), Zipf targets (hot dW rows), V tail."""
    inp = synth.make_inputs(1000, 200, 5000, seed=6, alpha=4.0, dist="zipf")
    budget = 4 << 20
    desc = slf.plan_describe(1000, 200, 5000, budget_bytes=budget, schedule="S")
    kv = dict(x.split("=") for x in desc.split())
    assert int(kv["n_chunks"]) > 2, desc
    check_against_oracle(slf, inp, reduction=reduction, budget=budget, schedule="S")


@pytest.mark.gpu
@pytest.mark.parametrize("reduction", ["mean", "none"])
def test_extended_chunks_parity_s(slf, reduction):
    """Schedule S with chunks extended into dhidden's unwritten rows: H/V large enough
    that ext rows fit (C = 256, chunks of 512 and 256 rows), ragged tail, Zipf targets; also dX only."""
    inp = synth.make_inputs(2000, 512, 1536, seed=16, alpha=4.0, dist="zipf")
    budget = 3 << 19
    desc = slf.plan_describe(2000, 512, 1536, budget_bytes=budget, schedule="S")
    assert "row_chunk=256" in desc, desc
    check_against_oracle(slf, inp, reduction=reduction, budget=budget, schedule="S")
    X, W, t = to_dev(inp, torch)
    _, dX1, _ = slf.lce_fwd_bwd(X, W, t, reduction=reduction, budget_bytes=budget, schedule="S",
                                need_dweight=False)
    _, dX2, _ = slf.lce_fwd_bwd(X, W, t, reduction=reduction, budget_bytes=budget, schedule="S")
    assert torch.equal(dX1, dX2)


@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("N,H,V", [(1, 8, 1), (1, 64, 300), (130, 136, 257), (257, 512, 4096)])
def test_small_edges(slf, N, H, V, sched):
    inp = synth.make_inputs(N, H, V, seed=N + V, alpha=2.0, ignore_frac=0.0 if N < 10 else 0.05)
    check_against_oracle(slf, inp, reduction="mean", schedule=sched)


@pytest.mark.parametrize("sched", SCHEDS)
def test_ignore_index_zero(slf, sched):
    inp = synth.make_inputs(300, 128, 1000, seed=3, ignore_index=0, alpha=2.0)
    check_against_oracle(slf, inp, reduction="mean", ignore_index=0, schedule=sched)


@pytest.mark.slow
@pytest.mark.parametrize("sched", SCHEDS)
def test_llama_head_reduced_n(slf, sched):
    """Full Llama-3.1-8B head (H=4096, V=128256) at N=1024: every element against the oracle."""
    inp = synth.make_config("llama8b", seed=21, alpha=4.0, dist="zipf", N=1024)
    ex, ew = check_against_oracle(slf, inp, reduction="mean", schedule=sched, budget=120 << 20)
    print(f"llama8b N=1024 {sched}: dX err {ex:.2e} dW err {ew:.2e}")


@pytest.mark.slow
@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("cfg", ["qwen7b", "mistral123b"])
def test_other_heads_reduced_n(slf, cfg, sched):
    inp = synth.make_config(cfg, seed=22, alpha=1.0, dist="uniform", N=1024)
    check_against_oracle(slf, inp, reduction="sum", scale=1.0 / 1024, schedule=sched, budget=120 << 20)


# ---- invariants ----------------------------------------------------------------------------------
def test_w_zero_closed_form(slf):
    inp = synth.make_config("tiny", seed=4)
    X, W, t = to_dev(inp, torch)
    W.zero_()
    loss, dX, dW = slf.lce_fwd_bwd(X, W, t, reduction="mean")
    torch.cuda.synchronize()
    assert float(loss) == pytest.approx(math.log(4096), rel=1e-6)
    assert torch.all(dX == 0)
    valid = inp.t != -100
    Xo = synth.bf16_bits_to_f64(inp.X)
    coef = 1.0 / valid.sum()
    ref = np.tile(coef * Xo[valid].sum(0) / 4096, (4096, 1))
    for i in np.nonzero(valid)[0]:
        ref[inp.t[i]] -= coef * Xo[i]
    assert rel_max_err(bf16_to_np64(dW), ref) < GRAD_TOL


@pytest.mark.parametrize("sched", SCHEDS)
def test_scale_linearity_and_determinism(slf, sched):
    inp = synth.make_inputs(700, 256, 3000, seed=9, alpha=3.0, dist="zipf")
    a = run_gpu(slf, inp, "mean", 1.0, budget=2 << 20, schedule=sched)
    b = run_gpu(slf, inp, "mean", 2.0, budget=2 << 20, schedule=sched)
    c = run_gpu(slf, inp, "mean", 1.0, budget=2 << 20, schedule=sched)
    assert float(a[0]) == float(b[0]) == float(c[0])
    assert torch.equal(a[1].float() * 2, b[1].float()) and torch.equal(a[2].float() * 2, b[2].float())
    assert torch.equal(a[1], c[1]) and torch.equal(a[2], c[2])


@pytest.mark.parametrize("sched", SCHEDS)
def test_ignored_rows_do_not_leak(slf, sched):
    inp = synth.make_inputs(400, 128, 2000, seed=10, alpha=2.0)
    a = run_gpu(slf, inp, "sum", schedule=sched)
    ign = inp.t == -100
    inp2 = synth.LCEInputs(**{**inp.__dict__})
    X2 = inp.X.copy()
    X2[ign] = synth.f32_to_bf16_bits(np.random.default_rng(0).standard_normal((ign.sum(), 128)).astype(np.float32) * 7)
    inp2.X = X2
    b = run_gpu(slf, inp2, "sum", schedule=sched)
    assert float(a[0]) == float(b[0])
    assert torch.equal(a[1][torch.from_numpy(~ign).cuda()], b[1][torch.from_numpy(~ign).cuda()])
    assert torch.equal(a[2].float().abs(), b[2].float().abs())


@pytest.mark.parametrize("sched", ["auto", "R"])
def test_status_counts(slf, sched):
    inp = synth.make_config("tiny", seed=1)
    X, W, t = to_dev(inp, torch)
    ws = slf.alloc_workspace(256, 512, 4096, X.device)
    loss, _, _ = slf.lce_fwd_bwd(X, W, t, workspace=ws, schedule=sched)
    bad, nv = slf.status(ws)
    assert bad == 0 and nv == 243
    t[5] = 4096
    loss, _, _ = slf.lce_fwd_bwd(X, W, t, workspace=ws, schedule=sched)
    bad, nv = slf.status(ws)
    assert bad == 1 and math.isnan(float(loss))


@pytest.mark.parametrize("sched", SCHEDS)
def test_all_ignored_mean(slf, sched):
    inp = synth.make_config("tiny", seed=2)
    inp.t[:] = -100
    loss, dX, dW = run_gpu(slf, inp, "mean", schedule=sched)
    assert float(loss) == 0.0 and torch.all(dX == 0) and torch.all(dW == 0)


# ---- split API, autograd, shard emulation --------------------------------------------------------
def test_split_matches_fused(slf):
    inp = synth.make_inputs(600, 256, 3000, seed=12, alpha=3.0)
    X, W, t = to_dev(inp, torch)
    loss_a, dX_a, dW_a = slf.lce_fwd_bwd(X, W, t, reduction="mean", schedule="R")
    loss_s, dX_s, dW_s = slf.lce_fwd_bwd(X, W, t, reduction="mean", schedule="S")
    assert abs(float(loss_s) - float(loss_a)) <= 1e-5 * abs(float(loss_a))
    assert rel_max_err(bf16_to_np64(dX_s), bf16_to_np64(dX_a)) < 1e-2
    assert rel_max_err(bf16_to_np64(dW_s), bf16_to_np64(dW_a)) < 1e-2
    loss_b, rs = slf.lce_fwd(X, W, t, reduction="mean")
    dX_b, dW_b = slf.lce_bwd(X, W, t, rs, 1.0)
    torch.cuda.synchronize()
    assert float(loss_a) == float(loss_b)
    assert torch.equal(dX_a, dX_b) and torch.equal(dW_a, dW_b)
    Xr = X.clone().requires_grad_(True)
    Wr = W.clone().requires_grad_(True)
    L = slf.LCEFunction.apply(Xr, Wr, t, -100, "mean")
    (3.0 * L).backward()
    assert torch.equal(Xr.grad.float(), dX_a.float() * 3) or rel_max_err(bf16_to_np64(Xr.grad), 3 * bf16_to_np64(dX_a)) < 1e-2


@pytest.mark.parametrize("g", [2, 3])
def test_vocab_shard_emulation(slf, g):
    """g vocab shards on one GPU through the split API (the multi-GPU seam): per-shard statistics,
    combine in shard order, per-shard backward with fp32 dX partials summed as an all-reduce would."""
    inp = synth.make_inputs(500, 256, 4100, seed=13, alpha=4.0, dist="zipf")
    X, W, t = to_dev(inp, torch)
    V = 4100
    bounds = [V * k // g for k in range(g + 1)]
    stats = torch.stack([slf.shard_stats(X, W[a:b].contiguous(), t, a) for a, b in zip(bounds[:-1], bounds[1:])])
    dX = torch.zeros(500, 256, dtype=torch.float32, device="cuda")
    dWs = []
    losses = []
    for k, (a, b) in enumerate(zip(bounds[:-1], bounds[1:])):
        loss, rs = slf.stats_combine(stats, t, a, b - a, V, reduction="mean")
        losses.append(float(loss))
        dXk, dWk = slf.lce_bwd(X, W[a:b].contiguous(), t, rs, 1.0, dhidden_fp32=True)
        dX += dXk
        dWs.append(dWk)
    torch.cuda.synchronize()
    assert len(set(losses)) == 1
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction="mean")
    assert_loss_close(losses[0], ref["loss"], "mean")
    assert rel_max_err(dX.cpu().numpy(), ref["dX"]) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(torch.cat(dWs)), ref["dW"]) <= GRAD_TOL
    ign = inp.t == -100
    assert np.all(dX.cpu().numpy()[ign] == 0)


# ---- full Llama-3.1-8B size, in the launch configuration bench.py times ---------------------------
@pytest.mark.slow
def test_llama_full_size_sampled(slf):
    inp = synth.make_config("llama8b", seed=0, alpha=1.0, dist="uniform")
    X, W, t = to_dev(inp, torch)
    loss_rows, dX, dW = slf.lce_fwd_bwd(X, W, t, reduction="none", scale=1.0)
    loss_m, dX_m, dW_m = slf.lce_fwd_bwd(X, W, t, reduction="mean")
    loss_r, dX_r, dW_r = slf.lce_fwd_bwd(X, W, t, reduction="mean", schedule="R")
    assert float(loss_r) == pytest.approx(float(loss_m), rel=1e-5)
    assert rel_max_err(bf16_to_np64(dW_m), bf16_to_np64(dW_r)) < 1e-2
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(inp.N, 48, replace=False))
    rows = np.concatenate([rows, np.nonzero(inp.t == -100)[0][:4]])
    Xo = synth.bf16_bits_to_f64(inp.X[rows])
    Wo = synth.bf16_bits_to_f64(inp.W)
    valid, nv, coef = oracle.coef_for(inp.t, -100, "mean", 1.0)
    l, lse, dXo, _ = oracle.rows(Xo, Wo, inp.t[rows].astype(np.int64), coef[rows])
    assert_loss_close(loss_rows.cpu().numpy()[rows], l, "none")
    assert rel_max_err(bf16_to_np64(dX_m)[rows], dXo) <= GRAD_TOL
    assert float(loss_m) == pytest.approx(float(loss_rows[torch.from_numpy(valid).cuda()].double().sum()) / nv, rel=1e-5)
    assert torch.isfinite(dW_m.float()).all()


@pytest.mark.parametrize("g,N,budget", [(2, 500, 1 << 21), (3, 700, 3 << 19)])
def test_vocab_shard_emulation_s(slf, g, N, budget):
    """Schedule S split for vocab shards, g shards emulated on one GPU: per chunk, every shard's
    statistics are stacked in rank order (the all-gather), each shard's fp32 dX partial is summed
    (the all-reduce) and finalised; dW stays per shard; the one-hot correction runs per shard."""
    from paper_2603_16428_b200 import lce as L
    V, H = 4100, 256
    inp = synth.make_inputs(N, H, V, seed=14, alpha=4.0, dist="zipf")
    X, W, t = to_dev(inp, torch)
    bounds = [V * k // g for k in range(g + 1)]
    shards = [L.SShard(X, W[a:b].contiguous(), t, a, V, reduction="mean", budget_bytes=budget)
              for a, b in zip(bounds[:-1], bounds[1:])]
    C, nch = shards[0].C, shards[0].n_chunks
    assert nch > 1 and all(s.C == C and s.n_chunks == nch for s in shards), (C, nch)
    dWs = [torch.empty(b - a, H, dtype=torch.bfloat16, device="cuda") for a, b in zip(bounds[:-1], bounds[1:])]
    dX = torch.empty(N, H, dtype=torch.bfloat16, device="cuda")
    for s in shards:
        s.begin()
    for ch in range(nch):
        r0, rows = shards[0].rows(ch)
        st = torch.stack([s.chunk_stats(ch) for s in shards])
        acc = torch.zeros(rows, H, dtype=torch.float32, device="cuda")
        for s, dWk in zip(shards, dWs):
            part = torch.empty(rows, H, dtype=torch.float32, device="cuda")
            s.chunk_bwd(ch, st, dX_chunk=part, dhidden_fp32=True, dW=dWk)
            acc += part
        L.dx_finalize_ptr(acc, shards[0].rowstat() + r0 * 16, dX[r0:r0 + rows])
    losses = []
    for s, dWk in zip(shards, dWs):
        lo = torch.empty(1, dtype=torch.float32, device="cuda")
        s.end(loss_out=lo, dW=dWk)
        losses.append(float(lo))
    torch.cuda.synchronize()
    assert len(set(losses)) == 1
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction="mean")
    assert_loss_close(losses[0], ref["loss"], "mean")
    assert rel_max_err(bf16_to_np64(dX), ref["dX"]) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(torch.cat(dWs)), ref["dW"]) <= GRAD_TOL
    assert np.all(dX.view(torch.int16).cpu().numpy()[inp.t == -100] == 0)


@pytest.mark.parametrize("sched", SCHEDS)
def test_vocab_sharded_module_world1(slf, sched):
    """VocabShardedLCE end to end with real NCCL collectives (world size 1 on this GPU)."""
    import os
    import torch.distributed as dist
    from paper_2603_16428_b200.sharded import VocabShardedLCE
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    inp = synth.make_inputs(900, 256, 5000, seed=15, alpha=4.0, dist="zipf")
    X, W, t = to_dev(inp, torch)
    m = VocabShardedLCE(5000, budget_bytes=6 << 20, schedule=sched)  # fits with the module's dX buffers
    loss, dX, dW = m.forward_backward(X, W, t, reduction="mean")
    torch.cuda.synchronize()
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction="mean")
    assert_loss_close(float(loss), ref["loss"], "mean")
    assert rel_max_err(bf16_to_np64(dX), ref["dX"]) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(dW), ref["dW"]) <= GRAD_TOL
    if sched == SCHEDS[-1]:
        dist.destroy_process_group()


@pytest.mark.parametrize("sched,red,pin", [("S", "mean", True), ("S", "none", False), ("R", "sum", True)])
def test_host_input_call_matches_device_call(slf, sched, red, pin):
    """slf_lce_fwd_bwd_host (host hidden/targets/loss, chunked copies overlapping the GEMMs) gives
    bit-identical results to the device call on the same inputs (same plan, same kernels)."""
    inp = synth.make_inputs(1100, 256, 3000, seed=23, alpha=4.0, dist="zipf")
    X, W, t = to_dev(inp, torch)
    budget = 2 << 20
    loss_d, dX_d, dW_d = slf.lce_fwd_bwd(X, W, t, reduction=red, scale=0.5, budget_bytes=budget, schedule=sched)
    Xh, th = X.cpu(), t.cpu()
    if pin:
        Xh, th = Xh.pin_memory(), th.pin_memory()
    loss_h, dX_h, dW_h = slf.lce_fwd_bwd_host(Xh, W, th, reduction=red, scale=0.5, budget_bytes=budget,
                                              schedule=sched)
    torch.cuda.synchronize()
    assert torch.equal(loss_h, loss_d.reshape(-1).cpu())
    assert torch.equal(dX_h, dX_d) and torch.equal(dW_h, dW_d)
    # a second call reuses the staging buffers after the first has finished reading them
    loss_h2, dX_h2, _ = slf.lce_fwd_bwd_host(Xh, W, th, reduction=red, scale=0.5, budget_bytes=budget,
                                             schedule=sched)
    torch.cuda.synchronize()
    assert torch.equal(loss_h2, loss_h) and torch.equal(dX_h2, dX_h)


def test_host_input_double_buffered_staging(slf):
    """Back-to-back host-input calls alternating two staging sets with no host synchronisation:
    step k+1's input copy may run under step k (the library waits per staging buffer for the last
    call that read it), and every step still computes on its own inputs (bit-identical to the
    device call on them)."""
    inp1 = synth.make_inputs(1100, 256, 3000, seed=24, alpha=4.0, dist="zipf")
    inp2 = synth.make_inputs(1100, 256, 3000, seed=25, alpha=1.0, dist="uniform")
    (X1, W, t1), (X2, _, t2) = to_dev(inp1, torch), to_dev(inp2, torch)
    budget = 2 << 20
    ref = {}
    for name, X, t in (("a", X1, t1), ("b", X2, t2)):
        ref[name] = slf.lce_fwd_bwd(X, W, t, budget_bytes=budget, schedule="S")
    host = {"a": (X1.cpu().pin_memory(), t1.cpu().pin_memory()), "b": (X2.cpu().pin_memory(), t2.cpu().pin_memory())}
    stg = [slf.HostStaging(1100, 256, X1.device) for _ in range(2)]
    ws = slf.alloc_workspace(1100, 256, 3000, X1.device, "S", budget)
    order = ["a", "b", "b", "a", "a", "b"]
    outs = []
    for i, name in enumerate(order):
        lh = torch.empty(1, dtype=torch.float32).pin_memory()
        dX = torch.empty_like(X1)
        dW = torch.empty_like(W)
        slf.lce_fwd_bwd_host(host[name][0], W, host[name][1], dX=dX, dW=dW, loss_host=lh, staging=stg[i % 2],
                             workspace=ws, budget_bytes=budget, schedule="S")
        outs.append((name, lh, dX, dW))
    torch.cuda.synchronize()
    for name, lh, dX, dW in outs:
        loss_d, dX_d, dW_d = ref[name]
        assert torch.equal(lh, loss_d.reshape(-1).cpu()), name
        assert torch.equal(dX, dX_d) and torch.equal(dW, dW_d), name


# ---- final RMSNorm + LCE ---------------------------------------------------
@pytest.mark.parametrize("sched,fused", [("R", False), ("S", False), ("S", True)])
@pytest.mark.parametrize("N,H,V,budget", [(300, 256, 3000, 0), (1000, 520, 4100, 0), (2000, 512, 1536, 3 << 20)])
def test_rmsnorm_lce_parity(slf, sched, fused, N, H, V, budget):
    """Final RMSNorm + LCE against oracle.rmsnorm_lce: the composition (R / S) and the fused call
    (slf_rmsnorm_lce_fwd_bwd; with a small budget: several extended chunks, so the per-chunk y
    buffer, the in-place dy -> dx and the chunk-ordered dg sum all run)."""
    inp = synth.make_inputs(N, H, V, seed=16, alpha=3.0, dist="zipf")
    x, W, t = to_dev(inp, torch)
    rng = np.random.default_rng(5)
    g_np = synth.f32_to_bf16_bits((1 + 0.2 * rng.standard_normal(H)).astype(np.float32))
    g = torch.from_numpy(g_np.view(np.int16)).view(torch.bfloat16).cuda()
    if fused and budget:
        assert "n_chunks=1 " not in slf.rmsnorm_lce_plan_describe(N, H, V, budget)
    loss, dx, dg, dW = slf.rmsnorm_lce_fwd_bwd(x, g, W, t, eps=1e-5, reduction="mean", schedule=sched, fused=fused,
                                               budget_bytes=budget)
    torch.cuda.synchronize()
    xo, Wo, to = oracle_inputs(inp)
    ref_loss, ref_dx, ref_dg, ref_dW = oracle.rmsnorm_lce(xo, synth.bf16_bits_to_f64(g_np), Wo, to, eps=1e-5,
                                                          reduction="mean")
    assert_loss_close(float(loss), ref_loss, "mean")
    assert rel_max_err(bf16_to_np64(dx), ref_dx) <= GRAD_TOL
    assert rel_max_err(dg.cpu().numpy(), ref_dg) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(dW), ref_dW) <= GRAD_TOL
    assert np.all(dx.view(torch.int16).cpu().numpy()[inp.t == -100] == 0)


@pytest.mark.parametrize("red", ["mean", "none"])
def test_rmsnorm_lce_fused_matches_composition(slf, red):
    """The fused call forms exactly the composition's y (same fp32 ops, same bf16 rounding) and runs
    the same chunk plan, so the per-tile statistics are the same bits; the loss agrees to fp32
    rounding (the two combine kernels merge a row's tile statistics in different fixed orders).
    dx, dW, dg agree to bf16 rounding: the fused call writes X' over its y buffer in every chunk
    (DESIGN.md §5d), the composition into dhidden's free rows where they fit, so its last chunk
    rescales the stash instead, and dg groups its fp32 row sums differently."""
    inp = synth.make_inputs(3000, 512, 2000, seed=27, alpha=3.0, dist="zipf")
    x, W, t = to_dev(inp, torch)
    g = (1 + 0.1 * torch.randn(512, generator=torch.Generator().manual_seed(1))).to(torch.bfloat16).cuda()
    a = slf.rmsnorm_lce_fwd_bwd(x, g, W, t, reduction=red, schedule="S", fused=True)
    b = slf.rmsnorm_lce_fwd_bwd(x, g, W, t, reduction=red, schedule="S", fused=False)
    torch.cuda.synchronize()
    la, lb = a[0].view(-1).double().cpu().numpy(), b[0].view(-1).double().cpu().numpy()
    assert np.max(np.abs(la - lb)) <= 1e-6 * np.max(np.abs(lb))
    assert rel_max_err(bf16_to_np64(a[1]), bf16_to_np64(b[1])) < 1e-2
    assert rel_max_err(bf16_to_np64(a[3]), bf16_to_np64(b[3])) < 1e-2
    assert rel_max_err(a[2].cpu().numpy(), b[2].cpu().numpy()) < 1e-2


@pytest.mark.slow
def test_rmsnorm_lce_fused_llama_reduced_n(slf):
    """Fused RMSNorm + LCE at the Llama-3.1-8B head (H=4096, V=128256), N=1024, a budget forcing
    several chunks: every element of loss, dx, dg, dW against oracle.rmsnorm_lce."""
    N, H, V = 1024, 4096, 128256
    budget = 90 << 20
    desc = slf.rmsnorm_lce_plan_describe(N, H, V, budget)
    assert "n_chunks=1 " not in desc, desc
    inp = synth.make_config("llama8b", seed=28, alpha=4.0, dist="zipf", N=N)
    x, W, t = to_dev(inp, torch)
    rng = np.random.default_rng(6)
    g_np = synth.f32_to_bf16_bits((1 + 0.2 * rng.standard_normal(H)).astype(np.float32))
    g = torch.from_numpy(g_np.view(np.int16)).view(torch.bfloat16).cuda()
    loss, dx, dg, dW = slf.rmsnorm_lce_fwd_bwd(x, g, W, t, reduction="mean", budget_bytes=budget)
    torch.cuda.synchronize()
    xo, Wo, to = oracle_inputs(inp)
    ref_loss, ref_dx, ref_dg, ref_dW = oracle.rmsnorm_lce(xo, synth.bf16_bits_to_f64(g_np), Wo, to, eps=1e-5,
                                                          reduction="mean")
    assert_loss_close(float(loss), ref_loss, "mean")
    assert rel_max_err(bf16_to_np64(dx), ref_dx) <= GRAD_TOL
    assert rel_max_err(dg.cpu().numpy(), ref_dg) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(dW), ref_dW) <= GRAD_TOL
    print(f"fused rmsnorm+lce llama8b N={N} [{desc}]")


# ---- gradient accumulation and the fused autograd function ----------------
@pytest.mark.parametrize("sched", SCHEDS)
def test_accumulate_dw(slf, sched):
    """Two micro-batches with accumulate_dw equal the sum of the two separate dW (bf16 tolerance)."""
    a = synth.make_inputs(600, 256, 3000, seed=17, alpha=3.0)
    b = synth.make_inputs(600, 256, 3000, seed=18, alpha=3.0)
    Xa, W, ta = to_dev(a, torch)
    Xb, _, tb = to_dev(b, torch)
    _, _, dWa = slf.lce_fwd_bwd(Xa, W, ta, reduction="sum", schedule=sched, budget_bytes=2 << 20)
    _, _, dWb = slf.lce_fwd_bwd(Xb, W, tb, reduction="sum", schedule=sched, budget_bytes=2 << 20)
    acc = dWa.clone()
    loss = torch.empty(1, dtype=torch.float32, device="cuda")
    dX = torch.empty_like(Xb)
    slf.lce_fwd_bwd(Xb, W, tb, reduction="sum", schedule=sched, budget_bytes=2 << 20, out=(loss, dX, acc),
                    accumulate_dw=True)
    torch.cuda.synchronize()
    ref = bf16_to_np64(dWa) + bf16_to_np64(dWb)
    assert rel_max_err(bf16_to_np64(acc), ref) < 1e-2


def test_fused_autograd_function(slf):
    inp = synth.make_inputs(500, 256, 3000, seed=19, alpha=3.0)
    X, W, t = to_dev(inp, torch)
    Xr = X.clone().requires_grad_(True)
    Wr = W.clone().requires_grad_(True)
    L = slf.LCEFunctionFused.apply(Xr, Wr, t, -100, "mean")
    (0.5 * L).backward()
    torch.cuda.synchronize()
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction="mean", scale=0.5)
    assert_loss_close(float(L.detach()), ref["loss"], "mean")
    assert rel_max_err(bf16_to_np64(Xr.grad), ref["dX"]) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(Wr.grad), ref["dW"]) <= GRAD_TOL


# ---- every BASELINE config at full size, in bench.py's launch configuration (sampled rows) --------
@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["llama8b", "qwen7b", "llama70b", "mistral123b"])
def test_full_size_sampled_rows_all_configs(slf, cfg):
    """Per-row loss and dX on 32 sampled rows (incl. ignored ones) at the config's full N, H, V with
    the default schedule and budget; run-to-run bit-identical outputs (determinism, p10)."""
    inp = synth.make_config(cfg, seed=1, alpha=1.0, dist="uniform")
    X, W, t = to_dev(inp, torch)
    loss_rows, dX, dW = slf.lce_fwd_bwd(X, W, t, reduction="none", scale=1.0)
    l2, dX2, dW2 = slf.lce_fwd_bwd(X, W, t, reduction="none", scale=1.0)
    torch.cuda.synchronize()
    assert torch.equal(loss_rows, l2) and torch.equal(dX, dX2) and torch.equal(dW, dW2)
    del l2, dX2, dW2
    rng = np.random.default_rng(3)
    rows = np.sort(np.concatenate([rng.choice(inp.N, 28, replace=False), np.nonzero(inp.t == -100)[0][:4]]))
    Xo = synth.bf16_bits_to_f64(inp.X[rows])
    Wo = synth.bf16_bits_to_f64(inp.W)
    valid, nv, coef = oracle.coef_for(inp.t, -100, "none", 1.0)
    l, lse, dXo, _ = oracle.rows(Xo, Wo, inp.t[rows].astype(np.int64), coef[rows])
    assert_loss_close(loss_rows.cpu().numpy()[rows], l, "none")
    assert rel_max_err(bf16_to_np64(dX)[rows], dXo) <= GRAD_TOL
    assert np.all(dX[torch.from_numpy(inp.t == -100).cuda()].view(torch.int16).cpu().numpy() == 0)


# (full-size dW rows of every head: tests/test_gpu_heads.py::test_full_size_dw_and_dx_rows)


# ---- vocab-sharded call with in-library collectives (slf_lce_fwd_bwd_sharded) ---------------------
@pytest.mark.parametrize("red,ign", [("mean", -100), ("none", -100), ("sum", 0)])
def test_native_sharded_nccl_world1(slf, red, ign):
    """The library's own NCCL communicator (dlopen'ed NCCL, comm stream + events) at world size 1:
    the whole sharded orchestration runs, with 1-rank collectives."""
    inp = synth.make_inputs(900, 256, 5000, seed=16, alpha=4.0, dist="zipf", ignore_index=ign)
    X, W, t = to_dev(inp, torch)
    comm = slf.Comm.nccl(slf.comm_unique_id(), 0, 1, torch.cuda.current_device())
    try:
        loss, dX, dW = slf.lce_fwd_bwd_sharded(X, W, t, 5000, comm, ignore_index=ign, reduction=red,
                                               budget_bytes=6 << 20)
        for mode in (1, 3):  # P2P statistics exchange, then also the dX exchange kernel (self only)
            comm.set_p2p(mode)
            lp, dXp, dWp = slf.lce_fwd_bwd_sharded(X, W, t, 5000, comm, ignore_index=ign, reduction=red,
                                                   budget_bytes=6 << 20)
            torch.cuda.synchronize()
            assert comm.p2p_timeouts() == 0
            assert torch.equal(dX.view(torch.int16), dXp.view(torch.int16)), mode
            assert torch.equal(dW.view(torch.int16), dWp.view(torch.int16)), mode
            assert torch.equal(loss.view(-1), lp.view(-1)), mode
        comm.set_p2p(False)
        torch.cuda.synchronize()
        assert "n_chunks=1 " not in slf.sharded_plan_describe(900, 256, 5000, 1, 0, 6 << 20)
        # a second call on the same communicator (events / comm stream reused) is bit-identical
        loss2, dX2, dW2 = slf.lce_fwd_bwd_sharded(X, W, t, 5000, comm, ignore_index=ign, reduction=red,
                                                  budget_bytes=6 << 20)
        torch.cuda.synchronize()
    finally:
        comm.close()
    assert torch.equal(dX.view(torch.int16), dX2.view(torch.int16))
    assert torch.equal(dW.view(torch.int16), dW2.view(torch.int16))
    assert torch.equal(loss.view(-1), loss2.view(-1))
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, ignore_index=ign, reduction=red)
    assert_loss_close(loss.detach().cpu().numpy(), ref["loss"], red)
    assert rel_max_err(bf16_to_np64(dX), ref["dX"]) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(dW), ref["dW"]) <= GRAD_TOL
    assert np.all(dX.view(torch.int16).cpu().numpy()[inp.t == ign] == 0)


def _run_native_ranks(tmp_path, g, red, budget, extra=(), env_extra=None):
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **(env_extra or {}))
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native_sharded_worker.py")
    tmp_path.mkdir(parents=True, exist_ok=True)
    procs = [subprocess.Popen([sys.executable, worker, "--rank", str(r), "--world", str(g), "--out", str(tmp_path),
                               "--budget", str(budget), "--reduction", red, *extra], env=env)
             for r in range(g)]
    try:
        for p in procs:
            assert p.wait(timeout=600) == 0
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    return [np.load(tmp_path / f"rank{r}.npz") for r in range(g)]


@pytest.mark.parametrize("g,red,budget", [(2, "mean", 3 << 20), (3, "sum", 3 << 20), (2, "none", 4 << 20)])
def test_native_sharded_callbacks(slf, tmp_path, g, red, budget):
    """g ranks of the native sharded call as g processes on this GPU, collectives through a gloo
    callback transport (tests/native_sharded_worker.py): every rank returns the same loss and
    dhidden, the dW shards assemble the full dW, all against the oracle.  Then the same ranks with
    the per-chunk statistics exchanged by the P2P one-shot all-gather over CUDA IPC (NEXT-3; here
    between processes on one GPU), two calls on one communicator: bit-identical results."""
    res = _run_native_ranks(tmp_path / "cb", g, red, budget)
    inp = synth.make_inputs(900, 256, 5000, seed=21, alpha=4.0, dist="zipf")
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction=red)
    nch = int(str(res[0]["plan"]).split("chunks_with_dhidden=")[1].split()[0])  # extended chunks (§9)
    assert nch > 1
    # per chunk: one statistics all-gather and one dX all-reduce; per call: one all-reduce of the
    # rows' target logits when any chunk takes the per-row stash reference (it needs
    # room for X' in dhidden's later rows, so not at every shape)
    n_ref = int(res[0]["ar"]) - nch
    assert n_ref in (0, 1)
    if (g, red) == (2, "mean"):
        assert n_ref == 1  # this shape runs the per-row reference path across ranks
    for r in res:
        assert int(r["ag"]) == nch and int(r["ar"]) == nch + n_ref
        assert np.array_equal(r["loss"], res[0]["loss"]) and np.array_equal(r["dX"], res[0]["dX"])
    assert_loss_close(res[0]["loss"] if red == "none" else float(res[0]["loss"].reshape(-1)[0]), ref["loss"], red)
    tobf = lambda a: a.astype(np.int16).view(np.uint16).astype(np.uint32) << 16  # noqa: E731
    dX = tobf(res[0]["dX"]).view(np.float32).astype(np.float64)
    dW = np.concatenate([tobf(r["dW"]).view(np.float32).astype(np.float64) for r in res])
    assert [int(r["v0"]) for r in res] + [int(res[-1]["v1"])] == [5000 * k // g for k in range(g + 1)]
    assert rel_max_err(dX, ref["dX"]) <= GRAD_TOL
    assert rel_max_err(dW, ref["dW"]) <= GRAD_TOL
    assert np.all(res[0]["dX"][inp.t == -100] == 0)
    p2p = _run_native_ranks(tmp_path / "p2p", g, red, budget, ("--p2p", "1", "--calls", "2"))
    for a, b in zip(res, p2p):
        assert int(b["timeouts"]) == 0
        assert int(b["ag"]) == 0 and int(b["ar"]) == nch + n_ref  # statistics no longer go through the transport
        for k in ("loss", "dX", "dW"):
            assert np.array_equal(a[k], b[k]), k
    # statistics AND dX through the P2P exchanges (the dX exchange kernel: rank-order sum of the g
    # fp32 partials of this rank's row slice, bf16 rows stored into every rank's dhidden)
    px = _run_native_ranks(tmp_path / "p2pdx", g, red, budget, ("--p2p", "3", "--calls", "2"))
    for a, b in zip(res, px):
        assert int(b["timeouts"]) == 0
        # no per-chunk collective: the two 80-byte IPC address records (dX partials, dhidden) and the
        # per-call target-logit all-reduce
        assert int(b["ag"]) == 2 and int(b["ar"]) == n_ref
        assert np.array_equal(a["loss"], b["loss"]) and np.array_equal(a["dW"], b["dW"])
        assert np.array_equal(b["dX"], px[0]["dX"])  # every rank holds the same dhidden
        if g == 2:  # two partials: a + b in either order, bit-identical to the gloo sum
            assert np.array_equal(a["dX"], b["dX"])
    dXp = tobf(px[0]["dX"]).view(np.float32).astype(np.float64)
    assert rel_max_err(dXp, ref["dX"]) <= GRAD_TOL
    assert np.all(px[0]["dX"][inp.t == -100] == 0)
    if g == 2:  # GEMM launches on 140 of the SMs (8 left to the communicator): same tiles, same bits
        rs = _run_native_ranks(tmp_path / "rsv", g, red, budget, env_extra={"SLF_COMM_SMS": "8"})
        for a, b in zip(res, rs):
            for k in ("loss", "dX", "dW"):
                assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("g,V,red", [(2, 3000, "mean"), (3, 3001, "none")])
def test_native_sharded_extended_chunks(slf, tmp_path, g, V, red):
    """The sharded call with chunks extended into dhidden's unwritten rows (N=2000, H=512: 8 plain
    chunks become 6; V=3001 at g=3 makes the shards' stash pitches differ, and every rank must still
    cut the same chunks): gloo callback transport, then the P2P statistics + dX exchanges — loss,
    dhidden and dW bit-identical between the two for g=2 (two partials), against the oracle."""
    N, H, budget = 2000, 512, 3 << 20
    args = ("--N", str(N), "--H", str(H), "--V", str(V))
    # the dX partial in its dedicated workspace region (the dhidden-top placement has
    # its own test below), so the chunks are the workspace stash's, extended
    env = {"SLF_SHARD_PART": "region"}
    base = _run_native_ranks(tmp_path / "cb", g, red, budget, args, env_extra=env)
    px = _run_native_ranks(tmp_path / "p2p", g, red, budget, (*args, "--p2p", "3", "--calls", "2"), env_extra=env)
    descs = [str(r["plan"]) for r in base]
    nch = {int(d.split("chunks_with_dhidden=")[1].split()[0]) for d in descs}
    plain = int(descs[0].split("n_chunks=")[1].split()[0])
    assert len(nch) == 1 and nch.pop() < plain and "dx_partial=workspace" in descs[0], descs
    inp = synth.make_inputs(N, H, V, seed=21, alpha=4.0, dist="zipf")
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction=red)
    tobf = lambda a: a.astype(np.int16).view(np.uint16).astype(np.uint32) << 16  # noqa: E731
    for res in (base, px):
        for r in res:
            assert np.array_equal(r["loss"], res[0]["loss"]) and np.array_equal(r["dX"], res[0]["dX"])
        assert_loss_close(res[0]["loss"] if red == "none" else float(res[0]["loss"].reshape(-1)[0]), ref["loss"], red)
        assert rel_max_err(tobf(res[0]["dX"]).view(np.float32).astype(np.float64), ref["dX"]) <= GRAD_TOL
        dW = np.concatenate([tobf(r["dW"]).view(np.float32).astype(np.float64) for r in res])
        assert rel_max_err(dW, ref["dW"]) <= GRAD_TOL
        assert np.all(res[0]["dX"][inp.t == -100] == 0)
    if g == 2:
        for a, b in zip(base, px):
            for k in ("loss", "dX", "dW"):
                assert np.array_equal(a[k], b[k]), k


def test_native_sharded_p2p_dx_uneven_shards(slf, tmp_path):
    """P2P dX exchange when g does not divide V (V=32001, g=2: shards of 16000 / 16001 rows, so the
    ranks' workspace layouts differ by 8 KB before the fp32 partials): each rank must read its peers'
    partial buffers at THEIR offsets.  Bit-identical to the gloo all-reduce (two
    partials), and against the oracle."""
    V, budget = 32001, 20 << 20
    assert len({slf.sharded_workspace_bytes(900, 256, V, 2, r, budget) for r in (0, 1)}) == 2
    base = _run_native_ranks(tmp_path / "cb", 2, "mean", budget, ("--V", str(V)))
    px = _run_native_ranks(tmp_path / "p2p", 2, "mean", budget, ("--V", str(V), "--p2p", "3", "--calls", "2"))
    for a, b in zip(base, px):
        assert int(b["timeouts"]) == 0
        for k in ("loss", "dX", "dW"):
            assert np.array_equal(a[k], b[k]), k
    inp = synth.make_inputs(900, 256, V, seed=21, alpha=4.0, dist="zipf")
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction="mean")
    tobf = lambda a: a.astype(np.int16).view(np.uint16).astype(np.uint32) << 16  # noqa: E731
    assert_loss_close(float(px[0]["loss"].reshape(-1)[0]), ref["loss"], "mean")
    assert rel_max_err(tobf(px[1]["dX"]).view(np.float32).astype(np.float64), ref["dX"]) <= GRAD_TOL
    dW = np.concatenate([tobf(r["dW"]).view(np.float32).astype(np.float64) for r in px])
    assert rel_max_err(dW, ref["dW"]) <= GRAD_TOL


def test_lce_fwd_bwd_group_world1(slf):
    """slf.lce_fwd_bwd(..., group=WORLD, V_global=V): the SURVEY §8(b) Python form of the sharded
    call, over the library's own NCCL communicator for the group (world size 1 here)."""
    import os
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        inp = synth.make_inputs(700, 256, 4100, seed=17, alpha=4.0, dist="zipf")
        X, W, t = to_dev(inp, torch)
        loss, dX, dW = slf.lce_fwd_bwd(X, W, t, group=dist.group.WORLD, V_global=4100, budget_bytes=6 << 20)
        torch.cuda.synchronize()
        Xo, Wo, to = oracle_inputs(inp)
        ref = oracle.lce(Xo, Wo, to)
        assert_loss_close(float(loss), ref["loss"], "mean")
        assert rel_max_err(bf16_to_np64(dX), ref["dX"]) <= GRAD_TOL
        assert rel_max_err(bf16_to_np64(dW), ref["dW"]) <= GRAD_TOL
    finally:
        from paper_2603_16428_b200 import lce as L
        for c in L._COMMS.values():
            c.close()
        L._COMMS.clear()
        dist.destroy_process_group()


def test_no_device_allocation_in_call(slf):
    """the extra device memory of a step is exactly the caller's workspace — the
    library allocates no device memory in the call (cudaMemGetInfo unchanged, torch's allocator peak
    unchanged with every output preallocated), at the bench's Llama-3.1-8B shape, and the workspace
    is <= 5 % of the N*V*2 logits."""
    N, H, V = 16384, 4096, 128256
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.randn(N, H, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(V, H, device="cuda", generator=g) / 64).to(torch.bfloat16)
    t = torch.randint(0, V, (N,), device="cuda", generator=g, dtype=torch.int32)
    t[::20] = -100
    ws = slf.alloc_workspace(N, H, V, X.device)
    assert ws.numel() <= 0.05 * N * V * 2
    out = (torch.empty(1, device="cuda"), torch.empty_like(X), torch.empty_like(W))
    slf.lce_fwd_bwd(X, W, t, workspace=ws, out=out)  # warm-up: module loading, attribute setup
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    torch.cuda.reset_peak_memory_stats()
    peak0 = torch.cuda.max_memory_allocated()
    slf.lce_fwd_bwd(X, W, t, workspace=ws, out=out)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free1 == free0, (free0, free1)
    assert torch.cuda.max_memory_allocated() == peak0
    assert torch.isfinite(out[0]).all()


@pytest.mark.parametrize("red", ["mean", "sum", "none"])
@pytest.mark.parametrize("sched", SCHEDS)
def test_native_dp_world1(slf, red, sched):
    """slf_lce_fwd_bwd_dp over the library's NCCL communicator at world size 1 is exactly the fused
    call (the n_valid and loss all-reduces of one rank are identities)."""
    inp = synth.make_inputs(700, 256, 3000, seed=26, alpha=4.0, dist="zipf")
    X, W, t = to_dev(inp, torch)
    comm = slf.Comm.nccl(slf.comm_unique_id(), 0, 1, torch.cuda.current_device())
    try:
        ld, dXd, dWd = slf.lce_fwd_bwd_dp(X, W, t, comm, reduction=red, scale=0.5, sync_dweight=True,
                                          budget_bytes=2 << 20, schedule=sched)
        lf, dXf, dWf = slf.lce_fwd_bwd(X, W, t, reduction=red, scale=0.5, budget_bytes=2 << 20, schedule=sched)
        torch.cuda.synchronize()
    finally:
        comm.close()
    assert torch.equal(ld.reshape(-1), lf.reshape(-1))
    assert torch.equal(dXd, dXf) and torch.equal(dWd, dWf)


@pytest.mark.parametrize("g,red", [(2, "mean"), (3, "mean"), (2, "sum")])
def test_native_dp_callbacks(slf, tmp_path, g, red):
    """g ranks of slf_lce_fwd_bwd_dp as g processes on this GPU (gloo callback transport): each rank
    holds a contiguous token slice and the full W; the MEAN denominator is summed on the device
    across ranks, every rank returns the global loss; its dhidden rows and the sum of the ranks' dW
    partials match the oracle on the whole batch."""
    res = _run_native_ranks(tmp_path, g, red, 2 << 20, ("--mode", "dp"))
    inp = synth.make_inputs(900, 256, 5000, seed=21, alpha=4.0, dist="zipf")
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction=red)
    for r in res:
        assert np.array_equal(r["loss"], res[0]["loss"])
        assert int(r["ar"]) == (2 if red == "mean" else 1)  # n_valid limbs + loss (SUM: loss only)
    assert_loss_close(float(res[0]["loss"].reshape(-1)[0]), ref["loss"], red)
    tobf = lambda a: a.astype(np.int16).view(np.uint16).astype(np.uint32) << 16  # noqa: E731
    dX = np.concatenate([tobf(r["dX"]).view(np.float32).astype(np.float64) for r in res])
    assert [int(r["v0"]) for r in res] + [int(res[-1]["v1"])] == [900 * k // g for k in range(g + 1)]
    dW = sum(tobf(r["dW"]).view(np.float32).astype(np.float64) for r in res)
    assert rel_max_err(dX, ref["dX"]) <= GRAD_TOL
    assert rel_max_err(dW, ref["dW"]) <= GRAD_TOL
    assert np.all(np.concatenate([r["dX"] for r in res])[inp.t == -100] == 0)


@pytest.mark.parametrize("N,H,V,g", [(4096, 512, 3000, 2), (4096, 256, 3001, 3)])
def test_native_sharded_partial_placement(slf, tmp_path, N, H, V, g):
    """Where the fp32 dX partial lives: the top of dhidden's unwritten rows (the
    last chunks' partials in the workspace stash's tail) against the dedicated workspace region,
    each forced with SLF_SHARD_PART; gloo transport, then the P2P statistics + dX exchanges (peers
    read each chunk's partial at its placement); every rank identical; against the oracle."""
    budget = 3 << 20
    inp = synth.make_inputs(N, H, V, seed=21, alpha=4.0, dist="zipf")
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction="mean")
    tobf = lambda a: a.astype(np.int16).view(np.uint16).astype(np.uint32) << 16  # noqa: E731
    args = ("--N", str(N), "--H", str(H), "--V", str(V))
    for mode, word in (("top", "dhidden_top"), ("region", "workspace")):
        for tag, extra in (("cb", ()), ("p2p", ("--p2p", "3", "--calls", "2"))):
            res = _run_native_ranks(tmp_path / f"{mode}_{tag}", g, "mean", budget, (*args, *extra),
                                    env_extra={"SLF_SHARD_PART": mode})
            plan = str(res[0]["plan"])
            assert f"dx_partial={word}" in plan, plan
            if mode == "top":  # chunks of both kinds
                assert int(plan.split("top_chunks=")[1].split()[0]) >= 2, plan
                assert int(plan.split("tail_chunks=")[1].split()[0]) >= 1, plan
            for r in res:
                assert int(r["timeouts"]) == 0
                assert np.array_equal(r["loss"], res[0]["loss"]) and np.array_equal(r["dX"], res[0]["dX"])
            assert_loss_close(float(res[0]["loss"].reshape(-1)[0]), ref["loss"], "mean")
            assert rel_max_err(tobf(res[0]["dX"]).view(np.float32).astype(np.float64), ref["dX"]) <= GRAD_TOL
            dW = np.concatenate([tobf(r["dW"]).view(np.float32).astype(np.float64) for r in res])
            assert rel_max_err(dW, ref["dW"]) <= GRAD_TOL
            assert np.all(res[0]["dX"][inp.t == -100] == 0)


def _chunk_kinds(slf, N, H, V, g, budget):
    """Kinds of the sharded call's row chunks (slf_lce_sharded_chunk_table): 'ext' (partial at
    dhidden's top, extended stash), 'top', 'short' (top, fewer rows than C), 'tail' (partial in
    the workspace stash tail), 'region'."""
    C = int(slf.sharded_plan_describe(N, H, V, g, 0, budget).split("row_chunk=")[1].split()[0])
    kinds = set()
    for k in slf.sharded_chunk_table(N, H, V, g, 0, budget):
        if k["part_off"] >= 0:
            kinds.add("ext" if k["ext"] else ("short" if k["rows"] < C else "top"))
        else:
            kinds.add("tail" if k["part_off"] == -1 else "region")
    return kinds


@pytest.mark.parametrize("N,H,V,budget", [(5000, 512, 2000, 4 << 20), (6000, 256, 1000, 2 << 20)])
@pytest.mark.parametrize("red", ["mean", "none"])
@pytest.mark.parametrize("mode", [0, 3])
def test_native_sharded_all_chunk_kinds_world1(slf, N, H, V, budget, red, mode):
    """The native sharded call (NCCL, world 1; mode 3: P2P statistics + dX exchanges) at shapes whose
    chunk table has every kind of chunk — extended with the partial at dhidden's top, plain top,
    shortened top, and workspace-tail chunks — against the oracle."""
    assert {"ext", "short", "tail"} <= _chunk_kinds(slf, N, H, V, 1, budget)
    inp = synth.make_inputs(N, H, V, seed=37, alpha=4.0, dist="zipf")
    X, W, t = to_dev(inp, torch)
    comm = slf.Comm.nccl(slf.comm_unique_id(), 0, 1, torch.cuda.current_device())
    try:
        if mode:
            comm.set_p2p(mode)
        loss, dX, dW = slf.lce_fwd_bwd_sharded(X, W, t, V, comm, reduction=red, budget_bytes=budget)
        torch.cuda.synchronize()
        assert comm.p2p_timeouts() == 0
    finally:
        comm.close()
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction=red)
    assert_loss_close(loss.detach().cpu().numpy() if red == "none" else float(loss), ref["loss"], red)
    assert rel_max_err(bf16_to_np64(dX), ref["dX"]) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(dW), ref["dW"]) <= GRAD_TOL
    assert np.all(dX.view(torch.int16).cpu().numpy()[inp.t == -100] == 0)


@pytest.mark.parametrize("g,N,H,V,budget", [(2, 3000, 512, 4001, 2 << 20), (4, 3000, 512, 4001, 1 << 20)])
def test_native_sharded_all_chunk_kinds_multirank(slf, tmp_path, g, N, H, V, budget):
    """g = 2 / 4 ranks (processes on one GPU; V = 4001: uneven shards) at shapes whose
    chunk table mixes extended top, plain or shortened top, and workspace-tail chunks: gloo transport and P2P
    exchanges, every rank identical, against the oracle."""
    kinds = _chunk_kinds(slf, N, H, V, g, budget)
    assert {"ext", "tail"} <= kinds and kinds & {"top", "short"}, kinds
    inp = synth.make_inputs(N, H, V, seed=21, alpha=4.0, dist="zipf")
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction="mean")
    tobf = lambda a: a.astype(np.int16).view(np.uint16).astype(np.uint32) << 16  # noqa: E731
    args = ("--N", str(N), "--H", str(H), "--V", str(V))
    for tag, extra in (("cb", ()), ("p2p", ("--p2p", "3", "--calls", "2"))):
        res = _run_native_ranks(tmp_path / tag, g, "mean", budget, (*args, *extra))
        for r in res:
            assert int(r["timeouts"]) == 0
            assert np.array_equal(r["loss"], res[0]["loss"]) and np.array_equal(r["dX"], res[0]["dX"])
        assert_loss_close(float(res[0]["loss"].reshape(-1)[0]), ref["loss"], "mean")
        assert rel_max_err(tobf(res[0]["dX"]).view(np.float32).astype(np.float64), ref["dX"]) <= GRAD_TOL
        dW = np.concatenate([tobf(r["dW"]).view(np.float32).astype(np.float64) for r in res])
        assert rel_max_err(dW, ref["dW"]) <= GRAD_TOL


@pytest.mark.parametrize("N,H,V", [(1, 8, 3), (257, 16, 130), (600, 72, 1000)])
@pytest.mark.parametrize("mode", [0, 3])
def test_native_sharded_edges_world1(slf, N, H, V, mode):
    """The native sharded call at edge shapes (one token, tiny vocabulary, H not a multiple of 64,
    ragged last chunk), over NCCL (mode 0) and over the P2P exchanges (mode 3), against the oracle."""
    inp = synth.make_inputs(N, H, V, seed=31, alpha=4.0, dist="uniform", ignore_frac=0.2)
    X, W, t = to_dev(inp, torch)
    comm = slf.Comm.nccl(slf.comm_unique_id(), 0, 1, torch.cuda.current_device())
    try:
        if mode:
            comm.set_p2p(mode)
        loss, dX, dW = slf.lce_fwd_bwd_sharded(X, W, t, V, comm, reduction="mean", budget_bytes=2 << 20)
        torch.cuda.synchronize()
        assert comm.p2p_timeouts() == 0
    finally:
        comm.close()
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.lce(Xo, Wo, to, reduction="mean")
    if (inp.t != -100).any():
        assert_loss_close(float(loss), ref["loss"], "mean")
    assert rel_max_err(bf16_to_np64(dX), ref["dX"]) <= GRAD_TOL
    assert rel_max_err(bf16_to_np64(dW), ref["dW"]) <= GRAD_TOL


@pytest.mark.parametrize("V,v0,v1", [(3000, 0, 3000), (5000, 1234, 3900)])
def test_stats_epilogues_vs_oracle(slf, V, v0, v1):
    """L0 blocks: the per-shard row statistics (m, s, z_t, hit) from the schedule-R
    statistics epilogue (slf_lce_fwd_shard_stats) and from the schedule-S stash epilogue + shard
    merge (slf_lce_s_chunk_stats), against the oracle's fp64 shard statistics; m to fp32 rounding of
    the bf16-input dot products, s relatively, z_t and hit exactly where the target is in the shard."""
    from paper_2603_16428_b200 import lce as L
    N, H = 700, 256
    inp = synth.make_inputs(N, H, V, seed=33, alpha=4.0, dist="zipf")
    X, W, t = to_dev(inp, torch)
    Ws = W[v0:v1].contiguous()
    Xo, Wo, to = oracle_inputs(inp)
    ref = oracle.shard_stats(Xo, Wo[v0:v1], to, v0)
    m_ref, s_ref, z_ref = (np.asarray(a, dtype=np.float64) for a in ref[:3])
    loc = to - v0
    hit_ref = (to != -100) & (loc >= 0) & (loc < v1 - v0)
    st_r = slf.shard_stats(X, Ws, t, v0).cpu().numpy().astype(np.float64)
    sh = L.SShard(X, Ws, t, v0, V, budget_bytes=2 << 20)
    sh.begin()
    st_s = np.concatenate([sh.chunk_stats(ch).cpu().numpy() for ch in range(sh.n_chunks)]).astype(np.float64)
    torch.cuda.synchronize()
    assert sh.n_chunks > 1
    scale_z = np.max(np.abs(m_ref))
    for st in (st_r, st_s):
        assert np.max(np.abs(st[:, 0] - m_ref)) <= 1e-5 * scale_z
        assert np.max(np.abs(st[:, 1] - s_ref) / s_ref) <= 1e-4
        assert np.array_equal(st[:, 3] == 1.0, hit_ref)
        assert np.max(np.abs(st[hit_ref, 2] - z_ref[hit_ref])) <= 1e-5 * scale_z
        assert not st[~hit_ref, 2].any()


# ---- target CSR: bit-exact against a stable sort ------------------------------
@pytest.mark.parametrize("N,V,v0,Vl,dist,ign", [
    (1, 10, 0, 10, "uniform", 0.0), (1000, 5000, 0, 5000, "zipf", 0.05), (4097, 300, 0, 300, "zipf", 0.1),
    (16384, 128256, 0, 128256, "zipf", 0.05), (16384, 128256, 64128, 16032, "uniform", 0.05),
    (65536, 32768, 0, 32768, "zipf", 0.05), (20000, 7, 0, 7, "uniform", 0.3), (9000, 5000, 1234, 2000, "same", 0.05),
    (5000, 5000, 0, 5000, "ignored", 0.0)])
def test_target_csr_bit_exact(slf, N, V, v0, Vl, dist, ign):
    """offsets = exclusive scan of the in-shard target histogram, token_idx = the in-shard valid
    tokens ordered by (target, token index) — numpy's stable argsort — every entry bit-exact,
    including the hit-row count; hot Zipf rows, one repeated target, all ignored, tiny V."""
    if dist in ("same", "ignored"):
        t = np.full(N, v0 + 7 if dist == "same" else -100, dtype=np.int32)
        t[::20] = -100
    else:
        t = synth.make_targets(N, V, seed=N + Vl, dist=dist, ignore_frac=ign)
    td = torch.from_numpy(t).cuda()
    off, idx = slf.target_csr(td, Vl, vocab_start=v0)
    torch.cuda.synchronize()
    off, idx = off.cpu().numpy(), idx.cpu().numpy()
    loc = t.astype(np.int64) - v0
    sel = (t != -100) & (loc >= 0) & (loc < Vl)
    counts = np.bincount(loc[sel], minlength=Vl)
    ref_off = np.concatenate([[0], np.cumsum(counts)])
    n = int(sel.sum())
    tok = np.nonzero(sel)[0]
    ref_idx = tok[np.argsort(loc[sel], kind="stable")]
    assert np.array_equal(off[:Vl + 1], ref_off)
    assert off[Vl + 1] == int((counts > 0).sum())
    assert np.array_equal(idx[:n], ref_idx)


# ---- per-row stash reference: rows where it does not fit -------------------------
@pytest.mark.parametrize("alpha", [25.0, 60.0])
@pytest.mark.parametrize("red", ["mean", "none"])
def test_stash_reference_fallback_rows(slf, alpha, red):
    """Logit spread large enough that many rows have a row max far above the target logit (loss
    > 128 nats: the per-row reference would overflow) while others fit: those rows fall back to the
    in-place rescale tile by tile, in the same chunks as the rows that keep the reference.  Against
    the oracle; also bit-identical dX between the two chunk modes is NOT expected (different
    roundings), so each is checked against the oracle separately."""
    inp = synth.make_inputs(1000, 256, 5000, seed=34, alpha=alpha, dist="zipf")
    check_against_oracle(slf, inp, reduction=red, schedule="S", budget=4 << 20)
    X, W, t = to_dev(inp, torch)
    loss, dX, dW = slf.lce_fwd_bwd(X, W, t, reduction=red, schedule="S", budget_bytes=4 << 20)
    torch.cuda.synchronize()
    assert torch.isfinite(dX.float()).all() and torch.isfinite(dW.float()).all()


def test_interleaved_schedule_bit_identical(slf, tmp_path):
    """The experimental interleaved group schedule (SLF_INTERLEAVE=1: dX tiles in K segments with
    the dW tiles of each segment's vocabulary rows in between) accumulates every tile in
    the same K order, so loss, dX and dW are the same bits as under the default LPT schedule."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import synth, paper_2603_16428_b200 as slf
from gpu_util import to_dev
inp = synth.make_inputs(1500, 512, 6000, seed=35, alpha=4.0, dist='zipf')
X, W, t = to_dev(inp, torch)
l, dX, dW = slf.lce_fwd_bwd(X, W, t, budget_bytes=6 << 20, schedule='S')
torch.cuda.synchronize()
np.savez(sys.argv[2], l=l.cpu().numpy(), dX=dX.view(torch.int16).cpu().numpy(), dW=dW.view(torch.int16).cpu().numpy())
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("0", "1"):
        f = str(tmp_path / f"il{mode}.npz")
        env = dict(os.environ, SLF_INTERLEAVE=mode)
        subprocess.run([sys.executable, "-c", code, root, f], check=True, env=env, timeout=300)
        out[mode] = np.load(f)
    for k in ("l", "dX", "dW"):
        assert np.array_equal(out["0"][k], out["1"][k]), k


@pytest.mark.parametrize("case", ["multichunk", "fallback", "dx_only", "none"])
def test_inkernel_combine_bit_identical(slf, tmp_path, case):
    """The per-row combine run inside the group launch (default) against the separate
    combine launch (SLF_INKERNEL_COMBINE=0): the same arithmetic in the same order, so loss, dX and dW
    are the same bits — multi-chunk with extended chunks, rows that need the in-place rescale (the
    stash flags them and the dX tiles wait for the combine), a dX-only call, reduction 'none'."""
    import os
    import subprocess
    import sys
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import synth, paper_2603_16428_b200 as slf
from gpu_util import to_dev
case = sys.argv[3]
alpha = 60.0 if case == 'fallback' else 4.0
N, H, V = (1000, 256, 5000) if case == 'fallback' else (3000, 512, 6000)
inp = synth.make_inputs(N, H, V, seed=36, alpha=alpha, dist='zipf')
X, W, t = to_dev(inp, torch)
l, dX, dW = slf.lce_fwd_bwd(X, W, t, budget_bytes=4 << 20, schedule='S', reduction='none' if case == 'none' else 'mean',
                            need_dweight=case != 'dx_only')
torch.cuda.synchronize()
np.savez(sys.argv[2], l=l.cpu().numpy(), dX=dX.view(torch.int16).cpu().numpy(),
         dW=(dW.view(torch.int16).cpu().numpy() if dW is not None else np.zeros(1)))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("0", "1"):
        f = str(tmp_path / f"cj{mode}.npz")
        env = dict(os.environ, SLF_INKERNEL_COMBINE=mode)
        subprocess.run([sys.executable, "-c", code, root, f, case], check=True, env=env, timeout=300)
        out[mode] = np.load(f)
    for k in ("l", "dX", "dW"):
        assert np.array_equal(out["0"][k], out["1"][k]), k
    assert "n_chunks=1 " not in slf.plan_describe(3000, 512, 6000, "S", 4 << 20)
