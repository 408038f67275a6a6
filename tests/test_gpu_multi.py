"""2-GPU test of the partitioned feature store (§8(e)): ranks own node-ID ranges, rows of
arbitrary gids come back through owner bucketing + NCCL all-to-all + shard gather + unpack,
bit-exact against the generator's closed form; and one partitioned NC train step whose
all-reduced gradients equal the mean of the per-rank oracle gradients.
Skipped unless >= 2 GPUs are visible (run with `gpurun --gpus 2`)."""
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


def _worker(rank, world, port, out, feat_dtype):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{rank}"))
    import synth
    from paper_2406_06022_b200 import build
    build.build()
    from paper_2406_06022_b200.dist import FeatureExchange, allreduce_mean, balanced_bounds, rank_step
    from paper_2406_06022_b200.runtime import GraphStore, RGCNTrainer
    cfg = synth.with_dtype(synth.scaled(synth.mag(), 0.01, "mag_small"), feat_dtype)
    tdt = torch.bfloat16 if feat_dtype == "bf16" else torch.float32
    dev = f"cuda:{rank}"
    bounds = balanced_bounds(cfg.counts, world)
    shards = [synth.feature_rows(cfg, t, torch.arange(int(bounds[t][rank]), int(bounds[t][rank + 1]), device=dev),
                                 "torch", dev).to(tdt) for t in range(cfg.num_ntypes)]
    ex = FeatureExchange(cfg.counts, world, rank, shards, cfg.feat_dim)
    rng = np.random.default_rng(rank)
    gids = np.sort(rng.integers(0, cfg.num_nodes, 3000)).astype(np.int64)
    outt = torch.empty((len(gids), cfg.feat_dim), dtype=tdt, device=dev)
    ex.gather(torch.from_numpy(gids).to(dev), len(gids), outt)
    exp = np.concatenate([synth.feature_rows(cfg, int(np.searchsorted(cfg.node_off, g, side="right") - 1),
                                             [g - cfg.node_off[np.searchsorted(cfg.node_off, g, side="right") - 1]])
                          for g in gids])
    out["rows_ok%d" % rank] = bool(np.array_equal(outt.float().cpu().numpy(), exp))
    # partitioned NC step: CSC replicated, features partitioned
    st = GraphStore(cfg.counts, cfg.etype_src(), cfg.etype_dst(), dev)
    for r in range(cfg.num_etypes):
        s_, d_ = synth.etype_coo(cfg, r, backend="torch", device=dev)
        st.load_etype(r, s_, d_)
    st.feat_dim = cfg.feat_dim
    st.feat_dtype = tdt
    tr = RGCNTrainer(st, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_classes, synth.init_params(cfg),
                     synth.param_order(cfg), torch.from_numpy(synth.labels(cfg)),
                     int(cfg.node_off[cfg.target_ntype]), lr=cfg.lr, rng_seed=cfg.rng_seed)
    tr.exchange = ex
    step = rank_step(0, rank, world)
    tr.forward_backward(torch.from_numpy(synth.nc_seeds(cfg, step)).to(dev), step)
    allreduce_mean(tr.grad)
    torch.cuda.synchronize()
    out["grad%d" % rank] = tr.grad.cpu().numpy().copy()
    out["loss%d" % rank] = float(tr.loss.item())
    # peer mode: shards mapped over NVLink (CUDA IPC), rows read inside the kernels
    from paper_2406_06022_b200.dist import PeerFeatures
    st2 = GraphStore(cfg.counts, cfg.etype_src(), cfg.etype_dst(), dev)
    for r in range(cfg.num_etypes):
        s_, d_ = synth.etype_coo(cfg, r, backend="torch", device=dev)
        st2.load_etype(r, s_, d_)
    pf = PeerFeatures(st2, cfg.counts, world, rank, shards, cfg.feat_dim)
    g2 = st2.gather(torch.from_numpy(gids).to(dev)).float().cpu().numpy()
    out["peer_rows_ok%d" % rank] = bool(np.array_equal(g2, exp))
    tr2 = RGCNTrainer(st2, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_classes, synth.init_params(cfg),
                      synth.param_order(cfg), torch.from_numpy(synth.labels(cfg)),
                      int(cfg.node_off[cfg.target_ntype]), lr=cfg.lr, rng_seed=cfg.rng_seed)
    tr2.load_inputs(torch.from_numpy(synth.nc_seeds(cfg, step)).to(dev))
    tr2.capture(step0=step, ws=world, allreduce=lambda gr: allreduce_mean(gr))   # whole step in one graph
    tr2.replay()
    torch.cuda.synchronize()
    out["peer_grad%d" % rank] = tr2.pview("W1", "g").cpu().numpy().copy()
    out["peer_W1_%d" % rank] = tr2.pview("W1").cpu().numpy().copy()
    out["peer_loss%d" % rank] = float(tr2.loss.item())
    dist.barrier()
    del pf
    dist.destroy_process_group()


@pytest.mark.parametrize("feat_dtype", ["f32", "bf16"])
def test_two_gpu_partitioned_features(feat_dtype):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out, feat_dtype), nprocs=2, join=True)
    assert out["rows_ok0"] and out["rows_ok1"]
    import oracle
    import synth
    from paper_2406_06022_b200.dist import rank_step
    from tests._pair import close
    cfg = synth.with_dtype(synth.scaled(synth.mag(), 0.01, "mag_small"), feat_dtype)
    og = oracle.Graph(cfg)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    flats, losses, slW, slb = [], [], [], []
    from tests._pair import close_slack, relu_tie_slack
    for r in range(2):
        step = rank_step(0, r, 2)
        res = oracle.nc_step(og, params, synth.nc_seeds(cfg, step), synth.labels(cfg), step, cfg.rng_seed)
        flats.append(np.concatenate([res.grads[k].reshape(-1) for k in synth.param_order(cfg)]))
        losses.append(res.loss)
        sW, sb, _ = relu_tie_slack(res, cfg.num_etypes, 0)
        slW.append(sW)
        slb.append(sb)
    exp = np.mean(flats, axis=0)
    for r in range(2):
        close(out["loss%d" % r], losses[r], what=f"rank {r} loss")
    # layer 0 (ReLU) gets the mean of the ranks' ReLU-tie slack (R-relutie); the rest rtol only
    slack = np.zeros_like(exp)
    nW = slW[0].size
    slack[:nW] = (0.5 * (slW[0] + slW[1])).reshape(-1)
    slack[nW:nW + slb[0].size] = 0.5 * (slb[0] + slb[1])
    close_slack(out["grad0"], exp, slack, what="all-reduced grads")
    np.testing.assert_array_equal(out["grad0"], out["grad1"])
    # peer (NVLink) mode inside one captured CUDA graph incl. the NCCL all-reduce
    assert out["peer_rows_ok0"] and out["peer_rows_ok1"]
    for r in range(2):
        close(out["peer_loss%d" % r], losses[r], what=f"peer rank {r} loss")
    names = synth.param_order(cfg)
    shapes = {k: synth.init_params(cfg)[k].size for k in names}
    o = int(np.cumsum([0] + [shapes[k] for k in names])[names.index("W1")])
    expW1 = exp[o:o + shapes["W1"]].reshape(out["peer_grad0"].shape)
    close(out["peer_grad0"], expW1, what="peer all-reduced grad W1")
    np.testing.assert_array_equal(out["peer_W1_0"], out["peer_W1_1"])


def _emb_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{rank}"))
    import synth
    from paper_2406_06022_b200 import build
    build.build()
    from paper_2406_06022_b200.dist import PeerEmbedding, rank_step
    from paper_2406_06022_b200.runtime import RGCNTrainer
    from tests._pair import gpu_store
    cfg = synth.scaled(synth.tiny_enc(), 0.5, "tiny_enc_half")
    dev = f"cuda:{rank}"
    st = gpu_store(cfg, device=dev)
    tr = RGCNTrainer(st, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_classes, synth.init_params(cfg),
                     synth.param_order(cfg), torch.from_numpy(synth.labels(cfg)),
                     int(cfg.node_off[cfg.target_ntype]), lr=cfg.lr, rng_seed=cfg.rng_seed)
    emb_t = [t for t in range(cfg.num_ntypes) if not cfg.project[t]]
    pes = {}
    for t in emb_t:
        E = np.random.default_rng(100 + t).normal(scale=0.3, size=(cfg.counts[t], cfg.feat_dim)).astype(np.float32)
        pes[t] = PeerEmbedding(torch.from_numpy(E).to(dev), world, rank)
        tr.set_embedding(t, torch.from_numpy(E), lr=0.01, eps=1e-10, peers=pes[t])
    step = rank_step(0, rank, world)
    tr.forward_backward(torch.from_numpy(synth.nc_seeds(cfg, step)).to(dev), step)
    torch.cuda.synchronize()
    gid = tr.sampler.block(0).src_gid.cpu().numpy()
    out["gid%d" % rank] = gid
    out["H0_%d" % rank] = tr.H0[: len(gid)].cpu().numpy().copy()
    out["dH0_%d" % rank] = tr.dH0[: len(gid)].cpu().numpy().copy()
    tr._sparse_update()
    for t in emb_t:
        out["E%d_%d" % (t, rank)] = pes[t].gather_full().cpu().numpy()
        out["bits_clear%d_%d" % (t, rank)] = int(pes[t].bits.abs().sum().item()) == 0
    torch.cuda.synchronize()
    dist.barrier()
    del tr, pes
    dist.destroy_process_group()


def test_two_gpu_partitioned_embeddings():
    """Learnable tables partitioned over 2 GPUs (§8(f) f1 with §8(e); R-sparsedist): each rank's
    H0 rows are the table's rows read from their owners over NVLink, and after one sparse update
    (push over NVLink, barrier, owner Adagrad) every rank sees the table the oracle's
    sparse_adagrad_dist gives from the two ranks' dH0 rows."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    import torch.multiprocessing as mp
    import oracle
    import synth
    from tests._pair import close
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_emb_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    cfg = synth.scaled(synth.tiny_enc(), 0.5, "tiny_enc_half")
    for t in [t for t in range(cfg.num_ntypes) if not cfg.project[t]]:
        E0 = np.random.default_rng(100 + t).normal(scale=0.3, size=(cfg.counts[t], cfg.feat_dim))
        E0 = E0.astype(np.float32).astype(np.float64)
        rows_r, grads_r = [], []
        for r in range(2):
            gid = out["gid%d" % r]
            pos = np.nonzero((gid >= cfg.node_off[t]) & (gid < cfg.node_off[t + 1]))[0]
            assert len(pos) > 0
            assert np.array_equal(out["H0_%d" % r][pos], E0[gid[pos] - cfg.node_off[t]].astype(np.float32))
            rows_r.append(gid[pos] - cfg.node_off[t])
            grads_r.append(out["dH0_%d" % r][pos].astype(np.float64))
        E, S = E0.copy(), np.zeros_like(E0)
        oracle.sparse_adagrad_dist(E, S, rows_r, grads_r, 0.01, 1e-10)
        for r in range(2):
            assert out["bits_clear%d_%d" % (t, r)]
            close(out["E%d_%d" % (t, r)], E, what=f"Emb{t} after the partitioned update (rank {r})")
