"""GPU parity of the input encoder (§8(a) a6): projected bf16 feature rows
(tcgen05 bf16 MMAs with split weights) and frozen tables, through the full NC train step, against
the fp64 oracle (rtol 1e-5, R-tol), on a tiny case and a MAG240M-shaped case (768-d papers)."""
import numpy as np
import pytest

import oracle
import synth
from tests._pair import close, close_slack, dsrc_tie_slack, gpu_store, oracle_graph


def _enc_slack(og, cfg, res, params):
    """R-relutie through the encoder: layer 0's ambiguous ReLU units give dH0 a slack
    (dsrc_tie_slack), which reaches dWin_t as |X_t|^T slack over the rows of type t."""
    sl = dsrc_tie_slack(res, cfg.num_etypes, 0, params["W0"])
    gids = res.blocks[0].src_gid
    ty = og.type_of(gids)
    extra = {}
    for t in range(cfg.num_ntypes):
        if cfg.project[t]:
            rows = np.nonzero(ty == t)[0]
            X = oracle.input_rows(og, t, gids[rows] - cfg.node_off[t])
            extra[f"Win{t}"] = np.abs(X).T @ sl[rows]
    return sl, extra

pytestmark = pytest.mark.gpu

CASES = {
    "tiny_enc": lambda: synth.scaled(synth.tiny_enc(), 0.5, "tiny_enc_half"),
    "mag240m_small": lambda: synth.scaled(synth.mag240m(), 2e-4, "mag240m_small"),
}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2406_06022_b200 import build
    build.build()
    return torch


@pytest.mark.parametrize("case", list(CASES))
def test_encoder_step_parity(torch_cuda, case):
    import torch
    from tests.test_gpu_parity import _compare_blocks, _gpu_trainer, check_grads
    cfg = CASES[case]()
    st, og = gpu_store(cfg), oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    assert tr.enc_types == [0]
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    labels = synth.labels(cfg)
    for step in range(2):
        for k in synth.param_order(cfg):
            tr.pview(k).copy_(torch.from_numpy(params[k].astype(np.float32)))
        seeds = synth.nc_seeds(cfg, step)
        tr.forward_backward(torch.from_numpy(seeds).cuda(), step)
        torch.cuda.synchronize()
        res = oracle.nc_step(og, params, seeds, labels, step, cfg.rng_seed)
        _compare_blocks(cfg, st, tr.sampler, res.blocks)
        n0 = len(res.blocks[0].src_gid)
        close(tr.H0[:n0].cpu().numpy(), res.extra["ins"][0], what=f"{case} step {step} H0")
        sl, extra = _enc_slack(og, cfg, res, params)
        close_slack(tr.dH0[:n0].cpu().numpy(), res.extra["dH0"], sl, what=f"{case} step {step} dH0")
        for l in range(len(cfg.fanouts)):
            nd = len(res.blocks[l].dst_gid)
            close(tr.hout[l][:nd].cpu().numpy(), res.hs[l], what=f"{case} step {step} h{l}")
        close(tr.loss.cpu().numpy()[0], res.loss, what=f"{case} loss")
        check_grads(tr, res, cfg, step, extra)
        for k in synth.param_order(cfg):   # move the point between steps (oracle SGD-like nudge)
            params[k] = params[k] - 1e-2 * np.sign(res.grads[k])


def test_encoder_pipelined_graph(torch_cuda):
    """The encoder inside the double-buffered CUDA-graph pipeline (bench.py's path)."""
    import torch
    from tests.test_gpu_parity import _gpu_trainer, check_grads
    cfg = CASES["mag240m_small"]()
    st, og = gpu_store(cfg), oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    opt = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    dev_seeds = [torch.from_numpy(synth.nc_seeds(cfg, i)).cuda() for i in range(4)]
    tr.pipeline_start((dev_seeds[0],), 0)
    for step in range(3):
        for k in synth.param_order(cfg):
            tr.pview(k).copy_(torch.from_numpy(params[k].astype(np.float32)))
            tr.pview(k, "m").copy_(torch.from_numpy(opt[k]["m"].astype(np.float32)))
            tr.pview(k, "v").copy_(torch.from_numpy(opt[k]["v"].astype(np.float32)))
        tr.pipeline_step(dev_seeds[step + 1])
        tr.pipeline_sync()
        torch.cuda.synchronize()
        res = oracle.nc_step(og, params, synth.nc_seeds(cfg, step), synth.labels(cfg), step, cfg.rng_seed)
        close(tr.loss.cpu().numpy()[0], res.loss, what=f"pipelined enc step {step} loss")
        check_grads(tr, res, cfg, step, _enc_slack(og, cfg, res, params)[1])
        for k in synth.param_order(cfg):
            oracle.adam(params[k], res.grads[k], opt[k]["m"], opt[k]["v"], cfg.lr, step + 1)
