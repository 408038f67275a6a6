"""GPU parity of learnable sparse embeddings: table rows in H0, dH0 (the
table's sparse gradient), and the sparse Adagrad update of exactly the touched rows, against
the fp64 oracle through two train steps (eager and CUDA graph)."""
import numpy as np
import pytest

import oracle
import synth
from tests._pair import RTOL_F32, close, close_slack, gpu_store, oracle_graph
from tests.test_gpu_encoder import _enc_slack

pytestmark = pytest.mark.gpu
LR, EPS = 0.01, 1e-10


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2406_06022_b200 import build
    build.build()
    return torch


def _adagrad_interval(E, S, rows, g, tol):
    """Oracle sparse Adagrad for gradients anywhere in [g - tol, g + tol] (5 points): Adagrad's
    first steps are ~ -lr sign(g), ill-conditioned where |g| ~ 0 (as R-adamtol)."""
    outs = []
    for k in (-1.0, -0.5, 0.0, 0.5, 1.0):
        e, s = E.copy(), S.copy()
        oracle.sparse_adagrad(e, s, rows, g + k * tol, LR, EPS)
        outs.append(e[rows])
    outs = np.stack(outs)
    return outs.min(0), outs.max(0)


@pytest.mark.parametrize("use_graph", [False, True])
def test_sparse_embedding_steps(torch_cuda, use_graph):
    import torch
    from tests.test_gpu_parity import _gpu_trainer
    cfg = synth.scaled(synth.tiny_enc(), 0.5, "tiny_enc_half")
    st, og = gpu_store(cfg), oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    rng = np.random.default_rng(9)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    emb_t = [t for t in range(cfg.num_ntypes) if not cfg.project[t]]
    state = {}
    for t in emb_t:
        E = rng.normal(scale=0.3, size=(cfg.counts[t], cfg.feat_dim)).astype(np.float32)
        tr.set_embedding(t, torch.from_numpy(E), lr=LR, eps=EPS)
        params[f"Emb{t}"] = E.astype(np.float64)
        state[t] = np.zeros_like(params[f"Emb{t}"])
    labels = synth.labels(cfg)
    for step in range(2):
        for k in synth.param_order(cfg):     # dense params restart from the oracle's point
            tr.pview(k).copy_(torch.from_numpy(params[k].astype(np.float32)))
            tr.pview(k, "m").zero_()
            tr.pview(k, "v").zero_()
        tr.t = 0
        seeds = synth.nc_seeds(cfg, step)
        if use_graph and step == 1:
            tr.capture(step)
            tr.load_inputs(torch.from_numpy(seeds).cuda())
            tr.counters[1] = 0
            tr.replay()
        else:
            tr.train_step(torch.from_numpy(seeds).cuda(), step)
        torch.cuda.synchronize()
        res = oracle.nc_step(og, params, seeds, labels, step, cfg.rng_seed)
        n0 = len(res.blocks[0].src_gid)
        close(tr.H0[:n0].cpu().numpy(), res.extra["ins"][0], what=f"step {step} H0 (table rows)")
        sl, _ = _enc_slack(og, cfg, res, params)
        close_slack(tr.dH0[:n0].cpu().numpy(), res.extra["dH0"], sl, what=f"step {step} dH0")
        gr = oracle.emb_grads(og, params, res.blocks[0].src_gid, res.extra["dH0"])
        ty = og.type_of(res.blocks[0].src_gid)
        for t in emb_t:
            rows, g = gr[t]
            assert len(rows) > 0
            tol = RTOL_F32 * np.abs(g) + RTOL_F32 * np.abs(g).max() + sl[ty == t]
            lo, hi = _adagrad_interval(params[f"Emb{t}"], state[t], rows, g, tol)
            E_gpu = tr.emb[t][0].cpu().numpy().astype(np.float64)
            pslack = 1e-6 * np.abs(hi) + 1e-7
            got = E_gpu[rows]
            assert not ((got < lo - pslack) | (got > hi + pslack)).any(), f"step {step} Emb{t} rows"
            untouched = np.setdiff1d(np.arange(cfg.counts[t]), rows)
            assert np.array_equal(E_gpu[untouched], params[f"Emb{t}"][untouched].astype(np.float32)), \
                f"step {step}: untouched rows of Emb{t} moved"
            # continue both sides from the GPU's table / state (steps compared one at a time)
            params[f"Emb{t}"] = E_gpu.copy()
            state[t] = tr.emb[t][1].cpu().numpy().astype(np.float64)


def test_partitioned_embedding_two_ranks_one_gpu(torch_cuda):
    """R-sparsedist on one GPU: two samplers play two ranks, the table of ntype 0 is split in two
    shards (separate allocations, as two ranks would hold them); forward reads each input row
    from its owner's shard, both ranks push 1/2 of their dH0 rows into the owners' accumulators,
    each owner applies Adagrad.  Expected: oracle.sparse_adagrad_dist over the two ranks' rows,
    two steps (the second on the updated table)."""
    import ctypes as C
    import torch
    from paper_2406_06022_b200._lib import call
    from paper_2406_06022_b200.runtime import MiniBatchSampler
    cfg = synth.tiny()
    st = gpu_store(cfg)
    t, d, W = 0, 64, 2
    n = int(cfg.counts[t])
    bounds = np.array([0, 2077, n], np.int64)
    rng = np.random.default_rng(5)
    E_full = rng.normal(size=(n, d)).astype(np.float32)
    E = [torch.from_numpy(E_full[bounds[w]:bounds[w + 1]].copy()).cuda() for w in range(W)]
    S = [torch.zeros_like(e) for e in E]
    G = [torch.zeros_like(e) for e in E]
    bits = [torch.zeros((int(bounds[w + 1] - bounds[w]) + 31) // 32, dtype=torch.int32, device="cuda")
            for w in range(W)]
    ptrs = lambda ts: (C.c_void_p * W)(*[t_.data_ptr() for t_ in ts])
    bnd = bounds.ctypes.data_as(C.c_void_p)
    sms = [MiniBatchSampler(st, cfg.fanouts, max_seeds=cfg.batch) for _ in range(W)]
    E64, S64 = E_full.astype(np.float64), np.zeros((n, d))
    for step in range(2):
        rows_r, grads_r, dH0s = [], [], []
        E_cur = torch.cat(E).cpu().numpy()          # the sharded table as the GPU holds it
        for r, sm in enumerate(sms):
            sm.sample(torch.from_numpy(synth.nc_seeds(cfg, 2 * step + r)).cuda(), cfg.rng_seed, step)
            gid = sm.block(0).src_gid.cpu().numpy()
            pos = np.nonzero((gid >= cfg.node_off[t]) & (gid < cfg.node_off[t + 1]))[0]
            H0 = torch.zeros((sm.input_rows(), d), dtype=torch.float32, device="cuda")
            call("gsb_sparse_emb_fwd_peers", sm.h, C.c_void_p(sm.arena.data_ptr()), t, W, bnd, ptrs(E), d,
                 C.c_void_p(H0.data_ptr()), None)
            assert np.array_equal(H0.cpu().numpy()[pos], E_cur[gid[pos] - cfg.node_off[t]]), step
            dH0 = rng.normal(size=(sm.input_rows(), d)).astype(np.float32)
            dH0s.append(torch.from_numpy(dH0).cuda())
            rows_r.append(gid[pos] - cfg.node_off[t])
            grads_r.append(dH0[pos].astype(np.float64))
        for r, sm in enumerate(sms):
            call("gsb_sparse_emb_push", sm.h, C.c_void_p(sm.arena.data_ptr()), t, W, bnd, ptrs(G), ptrs(bits),
                 C.c_void_p(dH0s[r].data_ptr()), d, 1.0 / W, None)
        for w in range(W):
            call("gsb_sparse_adagrad_apply", C.c_void_p(E[w].data_ptr()), C.c_void_p(S[w].data_ptr()),
                 C.c_void_p(G[w].data_ptr()), C.c_void_p(bits[w].data_ptr()), int(bounds[w + 1] - bounds[w]), d,
                 LR, EPS, None)
        oracle.sparse_adagrad_dist(E64, S64, rows_r, grads_r, LR, EPS)
        got_E = torch.cat(E).cpu().numpy()
        got_S = torch.cat(S).cpu().numpy()
        close(got_S, S64, what=f"step {step} Adagrad state")
        close(got_E, E64, what=f"step {step} table")
        assert all(int(b.abs().sum()) == 0 for b in bits) and all(float(g.abs().sum()) == 0 for g in G)
