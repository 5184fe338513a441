"""World-size-2/3 CPU tests (gloo) of the vocab-sharded orchestration (paper_2603_16428_b200.sharded).

The CUDA kernels cannot run here, so the per-shard compute ops are replaced by float64 stand-ins
built on the oracle's plain definitions; what is under test is the host-side logic of the N>1
path: shard bounds, the rank-ordered all-gather of per-token statistics, the shard-order combine,
the fp32 all-reduce of dX partials and the locality of dW.  The result must equal the single-process
oracle on the full vocabulary.
"""
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2603_16428_b200.sharded import VocabShardedLCE, shard_bounds, token_bounds


def _fake_ops():
    def shard_stats(X, W_l, t, v0, ignore_index=-100, workspace=None, budget_bytes=0):
        m, s, zt = oracle.shard_stats(X.numpy(), W_l.numpy(), t.numpy(), v0, ignore_index)
        V_l = W_l.shape[0]
        tt = t.numpy()
        hit = (tt != ignore_index) & (tt - v0 >= 0) & (tt - v0 < V_l)
        return torch.from_numpy(np.stack([m, s, zt, hit.astype(np.float64)], axis=1))

    def stats_combine(allst, t, v0, V_l, V, ignore_index=-100, reduction="mean", scale=1.0, workspace=None):
        a = allst.numpy()
        lse, z = oracle.combine_shards([(a[k, :, 0], a[k, :, 1], a[k, :, 2]) for k in range(a.shape[0])])
        tt = t.numpy()
        valid, nv, coef = oracle.coef_for(tt, ignore_index, reduction, scale)
        l = np.where(valid, lse - z, 0.0)
        loss = l.sum() if reduction == "sum" else (l.sum() / nv if nv else 0.0)
        tloc = np.where(valid & (tt - v0 >= 0) & (tt - v0 < V_l), tt - v0, -1)
        return torch.tensor(loss), types.SimpleNamespace(lse=lse, coef=coef, tloc=tloc, valid=valid)

    def lce_bwd(X, W_l, t, rs, grad_scale, dhidden_fp32=True, workspace=None, budget_bytes=0, out=None):
        Z = X.numpy() @ W_l.numpy().T
        P = np.exp(Z - rs.lse[:, None])
        rows = np.nonzero(rs.tloc >= 0)[0]
        P[rows, rs.tloc[rows]] -= 1.0
        G = grad_scale * rs.coef[:, None] * P
        dx32, dW = out
        dx32.copy_(torch.from_numpy(G @ W_l.numpy()))
        dW.copy_(torch.from_numpy(G.T @ X.numpy()))
        return dx32, dW

    def dx_finalize(dx32, rs, out=None):
        r = dx32.clone()
        r[torch.from_numpy(~rs.valid)] = 0.0
        return r

    class FakeSShard:
        """float64 stand-in for lce.SShard (schedule S split API) on this rank's vocab shard: chunked
        rows of CHUNK, per-chunk shard statistics, shard-order merge, fp64 dX partial, dW (+)=."""
        CHUNK = 7

        def __init__(self, X, W_l, t, v0, V, ignore_index, reduction, scale, budget, workspace):
            self.X, self.W, self.t = X.numpy(), W_l.numpy(), t.numpy()
            self.v0, self.ign, self.red, self.scale = v0, ignore_index, reduction, scale
            self.N = self.X.shape[0]
            self.C = self.CHUNK
            self.n_chunks = (self.N + self.C - 1) // self.C
            self.valid, self.nv, self.coef = oracle.coef_for(self.t, ignore_index, reduction, scale)
            self.lrows = np.zeros(self.N)

        def rows(self, ch):
            r0 = ch * self.C
            return r0, min(self.C, self.N - r0)

        def begin(self, need_dweight=True):
            pass

        def chunk_stats(self, ch, out):
            r0, n = self.rows(ch)
            sl = slice(r0, r0 + n)
            m, s_, zt = oracle.shard_stats(self.X[sl], self.W, self.t[sl], self.v0, self.ign)
            loc = self.t[sl] - self.v0
            hit = (self.t[sl] != self.ign) & (loc >= 0) & (loc < self.W.shape[0])
            out.copy_(torch.from_numpy(np.stack([m, s_, zt, hit.astype(np.float64)], axis=1)))
            return out

        def chunk_bwd(self, ch, stats, dX_chunk=None, dhidden_fp32=True, dW=None, loss_rows=None):
            r0, n = self.rows(ch)
            sl = slice(r0, r0 + n)
            a = stats.numpy()
            lse, z = oracle.combine_shards([(a[k, :, 0], a[k, :, 1], a[k, :, 2]) for k in range(a.shape[0])])
            self.lrows[sl] = np.where(self.valid[sl], lse - z, 0.0)
            if loss_rows is not None:
                loss_rows[sl] = torch.from_numpy(self.lrows[sl])
            P = np.exp(self.X[sl] @ self.W.T - lse[:, None])
            loc = self.t[sl] - self.v0
            rr = np.nonzero(self.valid[sl] & (loc >= 0) & (loc < self.W.shape[0]))[0]
            P[rr, loc[rr]] -= 1.0
            G = self.coef[sl][:, None] * P
            dX_chunk.copy_(torch.from_numpy(G @ self.W))
            part = torch.from_numpy(G.T @ self.X[sl])
            if ch == 0:
                dW.copy_(part)
            else:
                dW.add_(part)

        def end(self, loss_out=None, dW=None):
            if loss_out is not None:
                tot = self.lrows.sum()
                loss_out[0] = tot if self.red == "sum" else (tot / self.nv if self.nv else 0.0)

    def dx_finalize_rows(sh, dx32, r0, out):
        r = dx32.clone()
        r[torch.from_numpy(~sh.valid[r0:r0 + dx32.shape[0]])] = 0.0
        out.copy_(r)
        return out

    return types.SimpleNamespace(shard_stats=shard_stats, stats_combine=stats_combine, lce_bwd=lce_bwd,
                                 dx_finalize=dx_finalize, SShard=FakeSShard, dx_finalize_rows=dx_finalize_rows)


def _fake_ops_r():
    """The R-seam-only stand-ins (no SShard): VocabShardedLCE falls back to schedule R."""
    o = _fake_ops()
    return types.SimpleNamespace(shard_stats=o.shard_stats, stats_combine=o.stats_combine, lce_bwd=o.lce_bwd,
                                 dx_finalize=o.dx_finalize)


def _worker(rank, world, port, N, H, V, red, q, sched="R"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        X = rng.standard_normal((N, H))
        W = rng.standard_normal((V, H)) * 3 / np.sqrt(H)
        t = rng.integers(0, V, N)
        t[rng.permutation(N)[:5]] = -100
        lce = VocabShardedLCE(V, ops=_fake_ops() if sched == "S" else _fake_ops_r(), schedule=sched)
        assert lce.schedule == sched
        v0, v1 = lce.v0, lce.v1
        loss, dX, dW = lce.forward_backward(torch.from_numpy(X), torch.from_numpy(W[v0:v1].copy()),
                                            torch.from_numpy(t), reduction=red, scale=0.5)
        q.put((rank, np.asarray(loss), dX.numpy(), dW.numpy(), v0, v1))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,red,sched", [(2, "mean", "R"), (3, "sum", "R"), (2, "mean", "S"), (3, "sum", "S"),
                                             (2, "none", "S")])
def test_vocab_sharded_orchestration(world, red, sched):
    """Both orchestrations (R: one all-gather + one all-reduce; S: per row chunk an all-gather of the
    chunk's statistics and an asynchronous, double-buffered all-reduce of its dX partial)."""
    N, H, V = 40, 16, 203
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, H, V, red, q, sched)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    X = rng.standard_normal((N, H))
    W = rng.standard_normal((V, H)) * 3 / np.sqrt(H)
    t = rng.integers(0, V, N)
    t[rng.permutation(N)[:5]] = -100
    ref = oracle.lce(X, W, t, reduction=red, scale=0.5)
    res.sort(key=lambda r: r[0])
    covered = []
    for rank, loss, dX, dW, v0, v1 in res:
        if red == "none":
            np.testing.assert_allclose(loss, ref["loss"], rtol=1e-12, atol=1e-14)
        else:
            assert float(loss) == pytest.approx(ref["loss"], rel=1e-12)
        np.testing.assert_allclose(dX, ref["dX"], rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(dW, ref["dW"][v0:v1], rtol=1e-10, atol=1e-14)
        covered.append((v0, v1))
    assert covered[0][0] == 0 and covered[-1][1] == V
    assert all(a[1] == b[0] for a, b in zip(covered[:-1], covered[1:]))


def test_shard_bounds():
    for V in (128256, 203, 8):
        for g in (1, 2, 3, 8):
            b = [shard_bounds(V, g, r) for r in range(g)]
            assert b[0][0] == 0 and b[-1][1] == V
            assert all(x[1] == y[0] for x, y in zip(b[:-1], b[1:]))
            sizes = [y - x for x, y in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


# The token-sharded (data-parallel) mode runs inside the library (slf_lce_fwd_bwd_dp: the global
# MEAN denominator is summed on the device); its multi-rank behaviour is tested on the GPU with g
# processes over a gloo callback transport (tests/test_gpu_parity.py::test_native_dp_callbacks).
