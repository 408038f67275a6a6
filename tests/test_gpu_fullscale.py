"""GPU parity at the bench configuration itself: the ogbn-mag-shaped graph at full size
(1.94M nodes, 36.8M stored edges, 128-d bf16 feature rows, fanouts [15, 10], batch 1024) run
exactly as bench.py times it (double-buffered pipeline, per-buffer CUDA graphs, fused
layer-0 gather) against the oracle on the same seeded inputs: blocks bit-exact, layer
outputs, loss and every gradient within rtol 1e-5 (R-tol, R-relutie)."""
import numpy as np
import pytest

import oracle
import synth
from tests._pair import close, gpu_store, oracle_graph
from tests.test_gpu_parity import _compare_blocks, _gpu_trainer, check_grads

pytestmark = pytest.mark.gpu


def test_mag_bf16_full_scale_pipelined_steps():
    import torch
    from paper_2406_06022_b200 import build
    build.build()
    cfg = synth.with_dtype(synth.mag(), "bf16")
    st = gpu_store(cfg)
    og = oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    train = synth.train_nodes(cfg)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    opt = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    labels = synth.labels(cfg)
    steps = [0, 5]          # batch indices (RNG step words) of the two computed batches
    seeds = [synth.nc_seeds(cfg, s, train) for s in steps + [9]]
    dev = [torch.from_numpy(s).cuda() for s in seeds]
    tr.pipeline_start((dev[0],), steps[0])
    for k, step in enumerate(steps):
        for name in synth.param_order(cfg):   # start from the oracle's state (fp32-rounded)
            tr.pview(name).copy_(torch.from_numpy(params[name].astype(np.float32)))
            tr.pview(name, "m").copy_(torch.from_numpy(opt[name]["m"].astype(np.float32)))
            tr.pview(name, "v").copy_(torch.from_numpy(opt[name]["v"].astype(np.float32)))
        tr.counters[0] = steps[k + 1] if k + 1 < len(steps) else 9   # step word of the batch sampled next
        tr.pipeline_step(dev[k + 1])
        tr.pipeline_sync()
        torch.cuda.synchronize()
        assert tr.sampler.poll_error() == 0
        res = oracle.nc_step(og, params, seeds[k], labels, step, cfg.rng_seed)
        _compare_blocks(cfg, st, tr.sampler, res.blocks)
        assert len(res.blocks[0].e_src_gid) > 200_000          # the full-size input block
        for l in range(len(cfg.fanouts)):
            nd = len(res.blocks[l].dst_gid)
            close(tr.hout[l][:nd].cpu().numpy(), res.hs[l], what=f"step {step} h{l}")
        close(tr.loss.cpu().numpy()[0], res.loss, what=f"step {step} loss")
        check_grads(tr, res, cfg, step)
        for name in synth.param_order(cfg):
            oracle.adam(params[name], res.grads[name], opt[name]["m"], opt[name]["v"], cfg.lr, k + 1)
