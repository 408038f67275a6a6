"""Multi-GPU test of the node-ID partitioned graph (§8(e) as north_star states it: "the graph
and node features are partitioned by node ID"; P:L86 sampling "on a distributed graph", P:L211
random partition; S:L240 edges owned by their dst's owner, S:L260 a worker reads only its own
partition's storage).  Every rank builds only the CSC shard of the dst nodes it owns
(gsb_csc_build_range) and its feature rows; the shards are mapped over NVLink (PeerCSC,
PeerFeatures) and the sampler reads remote segments from their owners.  Checked against the
oracle on the whole graph: every rank's blocks bit-exact (keyed draws, R-rng), the pipelined
CUDA-graph steps' losses, and the NCCL-mean gradients equal the mean of the per-rank oracle
gradients.  Runs at world = number of visible GPUs (2 or 4; `gpurun --gpus N`)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(name):
    import synth
    if name == "mag_small_bf16":
        return synth.with_dtype(synth.scaled(synth.mag(), 0.01, "mag_small"), "bf16")
    return synth.scaled(synth.synth_1b(), 0.01, "synth_small")


def _worker(rank, world, port, out, name, mode):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{rank}"))
    import synth
    from paper_2406_06022_b200 import build
    build.build()
    from paper_2406_06022_b200.dist import (FeatureExchange, PeerCSC, PeerFeatures, SampleExchange, allreduce_mean,
                                            balanced_bounds, rank_step)
    from paper_2406_06022_b200.runtime import GraphStore, RGCNTrainer
    cfg = _cfg(name)
    dev = f"cuda:{rank}"
    bounds = balanced_bounds(cfg.counts, world)
    st = GraphStore(cfg.counts, cfg.etype_src(), cfg.etype_dst(), dev)
    for r in range(cfg.num_etypes):
        s_, d_ = synth.etype_coo(cfg, r, backend="torch", device=dev)
        t = int(cfg.etypes[r].dst)
        st.load_etype_range(r, s_, d_, int(bounds[t][rank]), int(bounds[t][rank + 1]))
        del s_, d_
    out["local_edges%d" % rank] = sum(st.n_edges)
    csc = PeerCSC(st, world, rank, bounds, map_peers=(mode == "peer"))
    shards = [synth.feature_table(cfg, t, "torch", dev, lo=int(bounds[t][rank]), hi=int(bounds[t][rank + 1]))
              for t in range(cfg.num_ntypes)]
    if mode == "peer":
        pf = PeerFeatures(st, cfg.counts, world, rank, shards, cfg.feat_dim)
    else:                         # NCCL all-to-all of features (C4/C5)
        pf = FeatureExchange(cfg.counts, world, rank, shards, cfg.feat_dim)
        st.feat_dim = cfg.feat_dim
        st.feat_dtype = shards[0].dtype
    tr = RGCNTrainer(st, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_classes, synth.init_params(cfg),
                     synth.param_order(cfg), torch.from_numpy(synth.labels(cfg)),
                     int(cfg.node_off[cfg.target_ntype]), lr=cfg.lr, rng_seed=cfg.rng_seed)
    tr.fuse_gather = False        # unique input rows fetched over NVLink in the sample phase
    if mode == "nccl":            # frontier exchange C2/C3 at every hop; features C4/C5
        sx = SampleExchange(tr.sampler, world, rank, first_hop=1)
        tr.exchange = pf
    # eager step 0 (seeds of global batch rank_step(0, rank)), blocks + grads
    step = rank_step(0, rank, world)
    tr.forward_backward(torch.from_numpy(synth.nc_seeds(cfg, step)).to(dev), step)
    allreduce_mean(tr.grad)
    torch.cuda.synchronize()
    assert tr.sampler.poll_error() == 0
    for l in range(len(cfg.fanouts)):
        b = tr.sampler.block(l)
        out[f"blk{rank}_{l}"] = (b.dst_gid.cpu().numpy(), b.src_gid.cpu().numpy(), b.seg_ptr.cpu().numpy(),
                                 b.e_src_gid.cpu().numpy(), b.e_eid.cpu().numpy())
    out["grad%d" % rank] = tr.grad.cpu().numpy().copy()
    out["loss%d" % rank] = float(tr.loss.item())
    if mode == "nccl":
        out["xbytes%d" % rank] = sx.bytes_sent
    # the bench configuration: pipelined per-buffer CUDA graphs + NCCL mean after each compute
    # graph (nccl mode: eager sample phase with the host-synced exchanges, captured compute)
    ar = lambda g: allreduce_mean(g)
    seeds = [torch.from_numpy(synth.nc_seeds(cfg, rank_step(i, rank, world))).to(dev) for i in range(1, 4)]
    tr.pipeline_start((seeds[0],), rank_step(1, rank, world), ws=world, allreduce=ar)
    tr.pipeline_step(seeds[1])
    tr.pipeline_sync()
    torch.cuda.synchronize()
    assert tr.sampler.poll_error() == 0
    b = tr.sampler.block(0)
    out[f"pipe_blk{rank}"] = (b.src_gid.cpu().numpy(), b.e_eid.cpu().numpy())
    out["pipe_loss%d" % rank] = float(tr.loss.item())
    dist.barrier()
    if mode == "nccl":
        del sx
    del pf, csc
    dist.destroy_process_group()


@pytest.mark.parametrize("name,mode", [("mag_small_bf16", "peer"), ("synth_small", "peer"),
                                       ("mag_small_bf16", "nccl"), ("synth_small", "nccl")])
def test_partitioned_topology_multi_gpu(name, mode):
    """mode peer: shards mapped over NVLink, read by the kernels; mode nccl: no rank reads
    another's storage -- frontier requests / sampled edges (C2/C3) and feature rows (C4/C5) go
    through NCCL all-to-alls, the owners sample their requests."""
    import torch
    world = min(torch.cuda.device_count(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs (gpurun --gpus 2 or 4)")
    import torch.multiprocessing as mp
    import oracle
    import synth
    from paper_2406_06022_b200.dist import rank_step
    from tests._pair import close, close_slack, relu_tie_slack
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, name, mode), nprocs=world, join=True)
    cfg = _cfg(name)
    og = oracle.Graph(cfg)
    # every rank stored only its own dst ranges: the shards partition the edges
    assert sum(out["local_edges%d" % r] for r in range(world)) == sum(len(x) for x in og.indices)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    flats, slW, slb = [], [], []
    for r in range(world):
        step = rank_step(0, r, world)
        res = oracle.nc_step(og, params, synth.nc_seeds(cfg, step), synth.labels(cfg), step, cfg.rng_seed)
        for l, ob in enumerate(res.blocks):
            dst, src, seg, esg, eid = out[f"blk{r}_{l}"]
            assert np.array_equal(dst, ob.dst_gid) and np.array_equal(src, ob.src_gid), (r, l)
            assert np.array_equal(esg, ob.e_src_gid) and np.array_equal(eid, ob.e_eid), (r, l)
            assert seg[-1] == len(ob.e_src_gid)
        close(out["loss%d" % r], res.loss, what=f"rank {r} loss")
        flats.append(np.concatenate([res.grads[k].reshape(-1) for k in synth.param_order(cfg)]))
        sW, sb, _ = relu_tie_slack(res, cfg.num_etypes, 0)
        slW.append(sW)
        slb.append(sb)
        if mode == "nccl":
            assert out["xbytes%d" % r] > 0
        # pipelined step (global batch rank_step(1, r)) under the partitioned graph
        step1 = rank_step(1, r, world)
        ob1 = oracle.sample_blocks(og, synth.nc_seeds(cfg, step1), cfg.fanouts, cfg.rng_seed, step1)
        src1, eid1 = out[f"pipe_blk{r}"]
        assert np.array_equal(src1, ob1[0].src_gid) and np.array_equal(eid1, ob1[0].e_eid), r
    exp = np.mean(flats, axis=0)
    slack = np.zeros_like(exp)
    nW = slW[0].size
    slack[:nW] = np.mean(slW, axis=0).reshape(-1)
    slack[nW:nW + slb[0].size] = np.mean(slb, axis=0)
    close_slack(out["grad0"], exp, slack, what="all-reduced grads")
    for r in range(1, world):
        np.testing.assert_array_equal(out["grad0"], out["grad%d" % r])
