"""One-GPU check of the node-ID partitioned graph store (§8(e)): the CSC of
every etype is built as `world` shards over the dst ranges the ranks would own
(gsb_csc_build_range) and the feature table as `world` row ranges; all shards live on this GPU
and are registered through the same tables the multi-GPU path fills with IPC-mapped peers
(gsb_graph_set_csc_peers, gsb_graph_set_feature_peers).  The sampler then resolves every
segment and row through the owner lookup, exactly as across GPUs.  Blocks must equal the
whole-graph oracle's bit-exactly and the step's loss / gradients must match it, for world 2, 3,
4 and 8 (uneven ranges, empty ranges of small ntypes)."""
import ctypes as C

import numpy as np
import pytest

import oracle
import synth
from tests._pair import close, oracle_graph
from tests.test_gpu_parity import _compare_blocks, _gpu_trainer, check_grads

pytestmark = pytest.mark.gpu


def partitioned_store(cfg, world, dev="cuda"):
    import torch
    from paper_2406_06022_b200._lib import call
    from paper_2406_06022_b200.dist import balanced_bounds
    from paper_2406_06022_b200.runtime import GraphStore
    bounds = balanced_bounds(cfg.counts, world)
    st = GraphStore(cfg.counts, cfg.etype_src(), cfg.etype_dst(), dev)
    keep = []
    shards = {}
    totals = {}
    for r in range(cfg.num_etypes):
        s_, d_ = synth.etype_coo(cfg, r, backend="torch", device=dev)
        t = int(cfg.etypes[r].dst)
        for w in range(world):
            st.load_etype_range(r, s_, d_, int(bounds[t][w]), int(bounds[t][w + 1]))
            shards[(r, w)] = (st.indptr[r], st.indices[r], st.eid_base[r])
            totals[r] = totals.get(r, 0) + st.n_edges[r]
            keep += [st.indptr[r], st.indices[r]]
    nb = C.c_size_t()
    call("gsb_csc_peers_bytes", C.byref(nb))
    table = torch.zeros(int(nb.value), dtype=torch.uint8, device=dev)
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    for r in range(cfg.num_etypes):
        ip = (C.c_void_p * world)(*[shards[(r, w)][0].data_ptr() for w in range(world)])
        ix = (C.c_void_p * world)(*[shards[(r, w)][1].data_ptr() for w in range(world)])
        eb = (C.c_int64 * world)(*[shards[(r, w)][2] for w in range(world)])
        call("gsb_graph_set_csc_peers", st.h, C.c_void_p(table.data_ptr()), r, world, b.ctypes.data_as(C.c_void_p),
             ip, ix, eb, totals[r], None)
    from paper_2406_06022_b200.runtime import DTYPE_CODE
    for t in range(cfg.num_ntypes):
        rows = [synth.feature_table(cfg, t, "torch", dev, lo=int(bounds[t][w]), hi=int(bounds[t][w + 1]))
                for w in range(world)]
        keep += rows
        ptrs = (C.c_void_p * world)(*[x.data_ptr() if x.numel() else None for x in rows])
        bt = np.ascontiguousarray(bounds[t], dtype=np.int64)
        call("gsb_graph_set_feature_peers", st.h, t, world, bt.ctypes.data_as(C.c_void_p), ptrs, cfg.feat_dim,
             DTYPE_CODE[rows[0].dtype])
    st.feat_dim = cfg.feat_dim
    st.feat_dtype = torch.bfloat16 if cfg.feat_dtype == "bf16" else torch.float32
    st._keep = (keep, table)
    return st


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("fuse", [True, False])
def test_partitioned_store_single_gpu(world, fuse):
    import torch
    from paper_2406_06022_b200 import build
    build.build()
    cfg = synth.with_dtype(synth.scaled(synth.mag(), 0.01, "mag_small"), "bf16")
    st = partitioned_store(cfg, world)
    og = oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    tr.fuse_gather = fuse
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    for step in (0, 3):
        seeds = synth.nc_seeds(cfg, step)
        tr.forward_backward(torch.from_numpy(seeds).cuda(), step)
        torch.cuda.synchronize()
        assert tr.sampler.poll_error() == 0
        res = oracle.nc_step(og, params, seeds, synth.labels(cfg), step, cfg.rng_seed)
        _compare_blocks(cfg, st, tr.sampler, res.blocks)
        close(tr.loss.cpu().numpy()[0], res.loss, what=f"world {world} step {step} loss")
        check_grads(tr, res, cfg, step)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_partitioned_rows_and_segments(world):
    """Every node's feature row through the owner lookup equals the closed form, and every
    node's sampled neighbourhood (fanout ALL) equals the whole-graph oracle's: the shard tables
    alone, before any layer."""
    import torch
    from paper_2406_06022_b200 import build
    from paper_2406_06022_b200.runtime import MiniBatchSampler
    build.build()
    cfg = synth.with_dtype(synth.scaled(synth.mag(), 0.01, "mag_small"), "bf16")
    st = partitioned_store(cfg, world)
    gids = torch.arange(cfg.num_nodes, dtype=torch.int64, device="cuda")
    rows = st.gather(gids).float().cpu().numpy()
    og = oracle_graph(cfg)
    assert np.array_equal(rows, oracle.gather(og, np.arange(cfg.num_nodes)))
    sm = MiniBatchSampler(st, [-1], max_seeds=cfg.num_nodes)
    for t in range(cfg.num_ntypes):
        seeds = np.arange(cfg.node_off[t], cfg.node_off[t + 1], dtype=np.int64)
        sm.sample(torch.from_numpy(seeds).cuda(), cfg.rng_seed, 0)
        assert sm.poll_error() == 0
        _compare_blocks(cfg, st, sm, oracle.sample_blocks(og, seeds, [-1], cfg.rng_seed, 0))
