"""Layer-Adam (include/slf_adam.h) against the fp64 oracle
(oracle/adam_oracle.py).  The host step runs on this CPU (``-m "not gpu"``); the device-fed
pipelined step needs a GPU.

Tolerance (fp32 arithmetic vs the fp64 definition): every fp32 operation rounds with relative error
u = 2^-24 and one step of the update is ~10 operations per element, so after T steps
max|p32 - p64| <= 16 u T (max|p| + sum_t max|dp_t|), max|m32 - m64| <= 16 u T max|g| and
max|v32 - v64| <= 16 u T max|g|^2 (a factor >= 1.6 over the operation count).  The bf16 parameter
copy is bit-exact RNE of the library's own fp32 master, and within one bf16 ulp of RNE(p64).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
U = 2.0 ** -24


@pytest.fixture(scope="module")
def adam():
    from paper_2603_16428_b200 import build
    build.build()
    from paper_2603_16428_b200 import adam as A
    return A


def _grads(n, T, seed):
    rng = np.random.default_rng(seed)
    gs = []
    for _ in range(T):
        g = (rng.standard_normal(n) * 10.0 ** rng.uniform(-5, -1, n)).astype(np.float32)
        gs.append(torch.from_numpy(g).bfloat16())
    return gs


def _run_host(A, p0, grads, kw, grad_scale):
    a = A.LayerAdam(p0.numel(), **kw)
    a.set_params(p0)
    outs = []
    for g in grads:
        out = torch.empty(p0.numel(), dtype=torch.bfloat16)
        a.step_host(g, grad_scale, out)
        outs.append(out)
    p, m, v, t = a.state()
    a.close()
    return p, m, v, t, outs


def _check(p, m, v, out, p0, grads, kw, grad_scale):
    T = len(grads)
    g64 = [g.double().numpy() for g in grads]
    pr, mr, vr, ups = oracle.adam_steps(p0.double().numpy(), g64, kw["lr"], kw["betas"][0], kw["betas"][1],
                                        kw["eps"], kw["weight_decay"], kw["adamw"], grad_scale)
    gmax = max(float(np.max(np.abs(g))) for g in g64) * abs(grad_scale)
    if not kw["adamw"]:
        gmax += kw["weight_decay"] * float(np.max(np.abs(pr)))
    ep = np.max(np.abs(p.double().numpy() - pr))
    assert ep <= 16 * U * T * (np.max(np.abs(pr)) + sum(ups)), ep
    assert np.max(np.abs(m.double().numpy() - mr)) <= 16 * U * T * gmax
    assert np.max(np.abs(v.double().numpy() - vr)) <= 16 * U * T * gmax ** 2
    bits = out.view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(bits, oracle.bf16_rne(p.numpy()))  # RNE of the library's own master, bit-exact
    ref = oracle.bf16_rne(pr).astype(np.int32)
    assert np.max(np.abs(bits.astype(np.int32) - ref)) <= 1  # one bf16 ulp (same sign: |p| >> ulp here)


CASES = [
    (dict(lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0, adamw=True), 1.0),
    (dict(lr=3e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1, adamw=True), 0.25),
    (dict(lr=1e-2, betas=(0.8, 0.99), eps=1e-6, weight_decay=0.01, adamw=False), 2.0),
]


@pytest.mark.parametrize("kw,gs", CASES)
@pytest.mark.parametrize("n", [1, 15, 4096 * 3 + 7, 100003])
def test_host_step_parity(adam, kw, gs, n):
    T = 5
    p0 = torch.from_numpy(np.random.default_rng(n).standard_normal(n).astype(np.float32))
    grads = _grads(n, T, seed=n + 1)
    p, m, v, t, outs = _run_host(adam, p0, grads, kw, gs)
    assert t == T
    _check(p, m, v, outs[-1], p0, grads, kw, gs)


def test_bf16_init_is_exact(adam):
    """set_params from bf16 widens exactly (the LM head's bf16 W as the first fp32 master)."""
    w = torch.randn(1000).bfloat16()
    a = adam.LayerAdam(1000)
    a.set_params(w)
    assert torch.equal(a.state()[0], w.float())


def test_scalar_and_avx512_paths_identical(adam, tmp_path):
    """The AVX-512 update and the scalar loop (SLF_ADAM_NO_AVX512=1, a fresh process) give the same
    bits: same operation order, no fused multiply-adds."""
    if adam.simd_width() != 16:
        pytest.skip("no AVX-512 on this host")
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "from paper_2603_16428_b200.adam import LayerAdam, simd_width\n"
        "rng = np.random.default_rng(5); n = 50021\n"
        "a = LayerAdam(n, lr=2e-3, weight_decay=0.05); a.set_params(torch.from_numpy(rng.standard_normal(n).astype(np.float32)))\n"
        "out = torch.empty(n, dtype=torch.bfloat16)\n"
        "for _ in range(4): a.step_host(torch.from_numpy(rng.standard_normal(n).astype(np.float32)).bfloat16(), 0.5, out)\n"
        "p, m, v, t = a.state(); np.savez(sys.argv[1], p=p.numpy(), m=m.numpy(), v=v.numpy(), o=out.view(torch.int16).numpy(), w=simd_width())\n"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for env_off in (False, True):
        f = str(tmp_path / f"r{int(env_off)}.npz")
        env = dict(os.environ)
        if env_off:
            env["SLF_ADAM_NO_AVX512"] = "1"
        subprocess.run([sys.executable, "-c", code, f], check=True, env=env)
        res.append(np.load(f))
    assert int(res[0]["w"]) == 16 and int(res[1]["w"]) == 1
    for k in ("p", "m", "v", "o"):
        assert np.array_equal(res[0][k], res[1][k]), k


def test_bad_config_rejected(adam):
    from paper_2603_16428_b200._lib import SlfError
    for kw in (dict(lr=-1.0), dict(betas=(1.0, 0.9)), dict(eps=0.0), dict(weight_decay=-0.1)):
        with pytest.raises(SlfError):
            adam.LayerAdam(10, **kw)


@pytest.mark.gpu
@pytest.mark.parametrize("n,chunk", [(100003, 1 << 14), (1 << 20, 0)])
def test_device_fed_step_matches_host_step(adam, n, chunk):
    """The pipelined device-fed step (chunked d2h, CPU update, h2d) gives exactly the host step's
    state and bf16 parameters, over three back-to-back steps (the second and third reuse the pinned
    staging while the previous copies may still be draining)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    kw = dict(lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, adamw=True)
    p0 = torch.randn(n).bfloat16()
    grads = _grads(n, 3, seed=9)
    p_h, m_h, v_h, _, outs = _run_host(adam, p0.float(), grads, kw, 0.5)
    a = adam.LayerAdam(n, chunk_elems=chunk, **kw)
    a.set_params(p0)
    param = p0.cuda()
    for g in grads:
        gd = g.cuda()
        a.step_device_async(gd, param, 0.5)
        a.wait()
    torch.cuda.synchronize()
    p, m, v, t = a.state()
    assert t == 3
    assert torch.equal(p, p_h) and torch.equal(m, m_h) and torch.equal(v, v_h)
    assert torch.equal(param.cpu().view(torch.int16), outs[-1].view(torch.int16))
    _check(p, m, v, outs[-1], p0.float(), grads, kw, 0.5)
