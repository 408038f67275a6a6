"""World-size-2 gloo tests (CPU) of the N>1 host path: gradient mean all-reduce and the
per-rank batch split.  Pins: S:L315 (grads g and -g average to zero), the mean over ranks
equals the single-process mean of the per-rank oracle gradients, and the
round-robin split covers consecutive global batches exactly once."""
import os

import numpy as np
import torch
import torch.multiprocessing as mp


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_06022_b200.dist import allreduce_mean, rank_step
    # g and -g -> zeros
    g = torch.arange(6, dtype=torch.float32) * (1 if rank == 0 else -1)
    allreduce_mean(g)
    out[f"sym{rank}"] = g.numpy().copy()
    # per-rank oracle gradients of a tiny NC step, averaged
    import oracle
    import synth
    cfg = synth.scaled(synth.tiny(), 0.2)
    og = oracle.Graph(cfg)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    step = rank_step(0, rank, world)
    res = oracle.nc_step(og, params, synth.nc_seeds(cfg, step), synth.labels(cfg), step, cfg.rng_seed)
    flat = torch.from_numpy(np.concatenate([res.grads[k].reshape(-1) for k in synth.param_order(cfg)]))
    allreduce_mean(flat)
    out[f"mean{rank}"] = flat.numpy().copy()
    dist.destroy_process_group()


def test_two_rank_gloo_allreduce_and_split():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert np.all(out["sym0"] == 0) and np.all(out["sym1"] == 0)
    # single-process reference: mean of the two ranks' oracle gradients
    import oracle
    import synth
    from paper_2406_06022_b200.dist import rank_step
    cfg = synth.scaled(synth.tiny(), 0.2)
    og = oracle.Graph(cfg)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    flats = []
    for r in range(world):
        step = rank_step(0, r, world)
        res = oracle.nc_step(og, params, synth.nc_seeds(cfg, step), synth.labels(cfg), step, cfg.rng_seed)
        flats.append(np.concatenate([res.grads[k].reshape(-1) for k in synth.param_order(cfg)]))
    exp = np.mean(flats, axis=0)
    np.testing.assert_allclose(out["mean0"], exp, rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(out["mean0"], out["mean1"])
    # round-robin split: steps 0..3 on 2 ranks cover global batches 0..7 exactly once
    seen = sorted(rank_step(s, r, world) for s in range(4) for r in range(world))
    assert seen == list(range(8))
