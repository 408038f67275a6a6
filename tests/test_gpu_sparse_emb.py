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
