"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Integer work (CSC, sampled blocks, relabel, gather) is bit-exact; floats are
within rtol 1e-5 (fp32, north_star) under |g-r| <= rtol|r| + rtol max|r|."""
import numpy as np
import pytest

import oracle
import synth
from tests._pair import close, close_slack, gpu_store, oracle_graph, relu_tie_slack

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2406_06022_b200 import build
    build.build()
    return torch


CASES = {
    "tiny": lambda: synth.tiny(),                                          # 64-d fp32 rows
    "mag_small": lambda: synth.scaled(synth.mag(), 0.01, "mag_small"),     # 128-d fp32
    "tiny_bf16": lambda: synth.with_dtype(synth.tiny(), "bf16"),           # 64-d bf16
    "mag_small_bf16": lambda: synth.with_dtype(synth.scaled(synth.mag(), 0.01, "mag_small"), "bf16"),
}


@pytest.fixture(scope="module", params=list(CASES))
def pair(request, torch_cuda):
    cfg = CASES[request.param]()
    return cfg, gpu_store(cfg), oracle_graph(cfg)


# ------------------------------------------------------------------ CSC + gather
def test_csc_bitexact(pair):
    cfg, st, og = pair
    for r in range(cfg.num_etypes):
        assert st.n_edges[r] == len(og.indices[r])
        assert np.array_equal(st.indptr[r].cpu().numpy(), og.indptr[r])
        assert np.array_equal(st.indices[r][:st.n_edges[r]].cpu().numpy(), og.indices[r])


def test_csc_keep_mask_bitexact(torch_cuda):
    cfg = synth.tiny()
    keep = {0: (np.arange(cfg.etypes[0].num_edges) % 3 != 0).astype(np.uint8)}
    st = gpu_store(cfg, keep=keep)
    og = oracle_graph(cfg, keep=keep)
    assert st.n_edges[0] == len(og.indices[0])
    assert np.array_equal(st.indptr[0].cpu().numpy(), og.indptr[0])
    assert np.array_equal(st.indices[0][:st.n_edges[0]].cpu().numpy(), og.indices[0])


def test_gather_bitexact(pair, torch_cuda):
    cfg, st, og = pair
    rng = np.random.default_rng(0)
    gids = np.concatenate([rng.integers(0, cfg.num_nodes, 5000), [0, cfg.num_nodes - 1]]).astype(np.int64)
    out = st.gather(torch_cuda.from_numpy(gids).cuda())
    assert out.dtype == (torch_cuda.bfloat16 if cfg.feat_dtype == "bf16" else torch_cuda.float32)
    assert np.array_equal(out.float().cpu().numpy(), oracle.gather(og, gids))


# ------------------------------------------------------------------ sampling
def _compare_blocks(cfg, st, sampler, oblocks):
    slots = st.slot_etypes()
    for l, ob in enumerate(oblocks):
        gb = sampler.block(l)
        assert np.array_equal(gb.dst_gid.cpu().numpy(), ob.dst_gid), f"layer {l} dst"
        assert np.array_equal(gb.src_gid.cpu().numpy(), ob.src_gid), f"layer {l} src"
        S = gb.num_slots
        seg = gb.seg_ptr.cpu().numpy()
        cnt = np.diff(seg).reshape(-1, S)
        t = np.searchsorted(cfg.node_off, ob.dst_gid, side="right") - 1
        exp = np.zeros_like(cnt)
        for j in range(len(ob.dst_gid)):
            for s, r in enumerate(slots[t[j]]):
                exp[j, s] = ob.seg_cnt[j, r]
        assert np.array_equal(cnt, exp), f"layer {l} segment counts"
        assert np.array_equal(gb.e_src_gid.cpu().numpy(), ob.e_src_gid), f"layer {l} edge src gid"
        assert np.array_equal(gb.e_eid.cpu().numpy(), ob.e_eid), f"layer {l} eid"
        assert np.array_equal(gb.e_src.cpu().numpy(), ob.e_src), f"layer {l} edge src row"


@pytest.mark.parametrize("fanouts", [None, [1, 3], [-1, 4], [32, 32]])
def test_sample_blocks_bitexact(pair, torch_cuda, fanouts):
    from paper_2406_06022_b200.runtime import MiniBatchSampler
    cfg, st, og = pair
    f = fanouts or cfg.fanouts
    if -1 in f and cfg.name != "tiny":
        pytest.skip("fanout ALL only on the tiny graph")
    sm = MiniBatchSampler(st, f, max_seeds=cfg.batch)
    for step in (0, 3):
        seeds = synth.nc_seeds(cfg, step)
        sm.sample(torch_cuda.from_numpy(seeds).cuda(), cfg.rng_seed, step)
        assert sm.poll_error() == 0
        ob = oracle.sample_blocks(og, seeds, f, cfg.rng_seed, step)
        _compare_blocks(cfg, st, sm, ob)


def test_sample_ragged_and_edge_cases(torch_cuda):
    """single seed, a seed of every type (mixed, type-grouped), zero-degree nodes."""
    from paper_2406_06022_b200.runtime import MiniBatchSampler
    cfg = synth.tiny()
    st, og = gpu_store(cfg), oracle_graph(cfg)
    indeg = {t: np.zeros(cfg.counts[t], np.int64) for t in range(cfg.num_ntypes)}
    for r in range(cfg.num_etypes):
        indeg[cfg.etypes[r].dst] += np.diff(og.indptr[r])
    iso = [int(np.nonzero(indeg[t] == 0)[0][0]) + int(cfg.node_off[t]) for t in range(cfg.num_ntypes)
           if (indeg[t] == 0).any()]
    cases = [np.array([7]), np.array(sorted([3, cfg.node_off[1] + 5, cfg.node_off[2] + 9])),
             np.array(sorted(set(iso + [11, 12])))]
    sm = MiniBatchSampler(st, cfg.fanouts, max_seeds=64)
    for i, seeds in enumerate(cases):
        seeds = seeds.astype(np.int64)
        sm.sample(torch_cuda.from_numpy(seeds).cuda(), 5, i)
        assert sm.poll_error() == 0
        _compare_blocks(cfg, st, sm, oracle.sample_blocks(og, seeds, cfg.fanouts, 5, i))


def test_sample_latched_errors(torch_cuda):
    from paper_2406_06022_b200.runtime import MiniBatchSampler
    cfg = synth.tiny()
    st = gpu_store(cfg)
    sm = MiniBatchSampler(st, cfg.fanouts, max_seeds=8)
    bad_group = np.array([cfg.node_off[1] + 1, 2], np.int64)       # type 1 before type 0
    sm.sample(torch_cuda.from_numpy(bad_group).cuda(), 1, 0)
    assert sm.poll_error() == 1
    from paper_2406_06022_b200 import _lib
    with pytest.raises(_lib.GsbError):
        sm.sample(torch_cuda.zeros(9, dtype=torch_cuda.int64).cuda(), 1, 0)   # over capacity: sync error


def test_sample_large_seed_set(torch_cuda):
    """Seed sets above 8192 take the grid-wide seed scan (sample.cu seed_scan_kernel): every
    node of the tiny graph as seeds (all ntypes, ragged type boundaries) matches the oracle's
    blocks bit for bit, and a grouping error deep inside the set is still latched."""
    from paper_2406_06022_b200.runtime import MiniBatchSampler
    cfg = synth.tiny()
    st, og = gpu_store(cfg), oracle_graph(cfg)
    n = int(cfg.node_off[-1])
    sm = MiniBatchSampler(st, cfg.fanouts, max_seeds=n)
    seeds = np.arange(n, dtype=np.int64)
    sm.sample(torch_cuda.from_numpy(seeds).cuda(), 5, 3)
    assert sm.poll_error() == 0
    _compare_blocks(cfg, st, sm, oracle.sample_blocks(og, seeds, cfg.fanouts, 5, 3))
    bad = seeds.copy()
    bad[9001] = int(cfg.node_off[1]) - 1          # a type-0 node after type-2 nodes
    sm.sample(torch_cuda.from_numpy(bad).cuda(), 5, 3)
    assert sm.poll_error() == 1


def test_sample_multi_tile_scans(torch_cuda):
    """The sampling scans at sizes where a block owns several tiles (sample.cu count_kernel /
    count_scan_kernel: more than 2368 x 256 segment entries; rank_sum / rank_scan: more than
    592 x 1024 bitmap words, i.e. > 19.4M nodes): a 24M-node graph with a small edge set and
    20k seeds, blocks bit-exact against the oracle, ragged last chunks included."""
    from paper_2406_06022_b200.runtime import GraphStore, MiniBatchSampler
    cfg = synth.Config(
        name="wide", ntypes=["A", "B"], counts=[24_000_003, 40_001],
        etypes=[synth.EType("r0", 0, 1, 300_000), synth.EType("r1", 1, 0, 300_000),
                synth.EType("r2", 1, 1, 200_000)],
        feat_dim=4, fanouts=[12, 15], batch=20_000, hidden=8, num_classes=2,
        target_ntype=1, gen_seed=2406060220 + 77)
    st = GraphStore(cfg.counts, cfg.etype_src(), cfg.etype_dst(), "cuda")
    for r in range(cfg.num_etypes):
        s_, d_ = synth.etype_coo(cfg, r, backend="torch", device="cuda")
        st.load_etype(r, s_, d_)
    og = oracle_graph(cfg)
    rng = np.random.default_rng(5)
    seeds = np.sort(rng.choice(cfg.counts[1], 20_000, replace=False)).astype(np.int64) + int(cfg.node_off[1])
    sm = MiniBatchSampler(st, cfg.fanouts, max_seeds=len(seeds))
    sm.sample(torch_cuda.from_numpy(seeds).cuda(), 9, 1)
    assert sm.poll_error() == 0
    _compare_blocks(cfg, st, sm, oracle.sample_blocks(og, seeds, cfg.fanouts, 9, 1))


def test_sample_deterministic(pair, torch_cuda):
    from paper_2406_06022_b200.runtime import MiniBatchSampler
    cfg, st, og = pair
    sm = MiniBatchSampler(st, cfg.fanouts, max_seeds=cfg.batch)
    seeds = torch_cuda.from_numpy(synth.nc_seeds(cfg, 1)).cuda()
    outs = []
    for _ in range(2):
        sm.sample(seeds, 9, 1)
        b = sm.block(0)
        outs.append((b.src_gid.cpu().numpy(), b.e_src.cpu().numpy(), b.e_eid.cpu().numpy()))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ full NC train step
def _gpu_trainer(cfg, st):
    import torch
    from paper_2406_06022_b200.runtime import RGCNTrainer
    return RGCNTrainer(st, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_classes, synth.init_params(cfg),
                       synth.param_order(cfg), torch.from_numpy(synth.labels(cfg)),
                       int(cfg.node_off[cfg.target_ntype]), lr=cfg.lr, rng_seed=cfg.rng_seed)


def check_grads(tr, res, cfg, step, extra_slack=None):
    """Gradients within rtol; the hidden ReLU layers' dW/db additionally get the slack of
    their ambiguous (|z| within tolerance of 0) activations (R-relutie); extra_slack adds
    per-parameter slack (e.g. input-encoder weights behind layer 0's ReLU)."""
    L = len(cfg.fanouts)
    slack = dict(extra_slack or {})
    for l in range(L - 1):
        sW, sb, _ = relu_tie_slack(res, cfg.num_etypes, l)
        slack[f"W{l}"], slack[f"b{l}"] = sW, sb
    for k in synth.param_order(cfg):
        g = tr.pview(k, "g").cpu().numpy()
        if k in slack:
            close_slack(g, res.grads[k], slack[k], what=f"step {step} grad {k}")
        else:
            close(g, res.grads[k], what=f"step {step} grad {k}")
    return slack


def _adam_interval(p, g, m, v, tol_g, lr, t):
    """Oracle Adam update evaluated for gradients across [g - tol_g, g + tol_g] (5 points):
    the interval of parameters consistent with the gradient tolerance (DESIGN.md R-adamtol;
    Adam's normalised step is ill-conditioned where |g| is near 0)."""
    outs = []
    for k in (-1.0, -0.5, 0.0, 0.5, 1.0):
        pp, mm, vv = p.copy(), m.copy(), v.copy()
        oracle.adam(pp, g + k * tol_g, mm, vv, lr, t)
        outs.append(pp)
    outs = np.stack(outs)
    return outs.min(0), outs.max(0), outs[2]


@pytest.mark.parametrize("fuse_gather", [True, False])
def test_nc_step_parity(pair, torch_cuda, fuse_gather):
    """3 steps; before each, the GPU state is set from the oracle's (fp32-rounded), then both
    run one full step: blocks, x0 bit-exact; activations, loss, grads within rtol; params
    after Adam inside the oracle's interval for gradients within the gradient tolerance."""
    import torch
    cfg, st, og = pair
    tr = _gpu_trainer(cfg, st)
    tr.fuse_gather = fuse_gather
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    opt = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    labels = synth.labels(cfg)
    rtol = 1e-5
    for step in range(3):
        for k in synth.param_order(cfg):
            tr.pview(k).copy_(torch.from_numpy(params[k].astype(np.float32)))
            tr.pview(k, "m").copy_(torch.from_numpy(opt[k]["m"].astype(np.float32)))
            tr.pview(k, "v").copy_(torch.from_numpy(opt[k]["v"].astype(np.float32)))
        tr.t = step
        seeds = synth.nc_seeds(cfg, step)
        tr.forward_backward(torch_cuda.from_numpy(seeds).cuda(), step)
        res = oracle.nc_step(og, params, seeds, labels, step, cfg.rng_seed)
        n0 = len(res.blocks[0].src_gid)
        if not fuse_gather:
            assert np.array_equal(tr.x0[:n0].float().cpu().numpy(), res.x0)
        for l in range(len(cfg.fanouts)):
            nd = len(res.blocks[l].dst_gid)
            close(tr.hout[l][:nd].cpu().numpy(), res.hs[l], what=f"step {step} h{l}")
        close(tr.loss.cpu().numpy()[0], res.loss, what="loss")
        slack = check_grads(tr, res, cfg, step)
        tr.optimizer_step()
        for k in synth.param_order(cfg):
            g = res.grads[k]
            tol_g = rtol * np.abs(g) + rtol * np.abs(g).max() + slack.get(k, 0.0)
            lo, hi, mid = _adam_interval(params[k], g, opt[k]["m"], opt[k]["v"], tol_g, cfg.lr, step + 1)
            gp = tr.pview(k).cpu().numpy().astype(np.float64)
            pslack = rtol * np.abs(mid) + rtol * np.abs(mid).max()
            bad = (gp < lo - pslack) | (gp > hi + pslack)
            assert not bad.any(), f"step {step} param {k}: {bad.sum()} outside the Adam interval"
            oracle.adam(params[k], g, opt[k]["m"], opt[k]["v"], cfg.lr, step + 1)


def test_adam_kernel_parity(torch_cuda):
    import ctypes as C
    import torch
    from paper_2406_06022_b200._lib import call
    rng = np.random.default_rng(3)
    n = 1000
    p0 = rng.standard_normal(n).astype(np.float32)
    p, m, v = (torch.from_numpy(x).cuda() for x in (p0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)))
    pd, md, vd = p0.astype(np.float64), np.zeros(n), np.zeros(n)
    for t in range(1, 4):
        g = rng.standard_normal(n).astype(np.float32)
        gt = torch.from_numpy(g).cuda()
        call("gsb_adam_step", C.c_void_p(p.data_ptr()), C.c_void_p(gt.data_ptr()), C.c_void_p(m.data_ptr()),
             C.c_void_p(v.data_ptr()), n, 0.01, 0.9, 0.999, 1e-8, t, None, None)
        oracle.adam(pd, g, md, vd, 0.01, t)
    torch.cuda.synchronize()
    close(p.cpu().numpy(), pd, what="adam")


def test_cuda_graph_replay_matches_oracle(torch_cuda):
    """A whole step captured once in a CUDA graph and replayed: the step word and Adam t
    advance on the device; the replayed step's blocks are bit-exact and its loss and
    gradients match the oracle (the graph path is the one bench.py times)."""
    import torch
    cfg = synth.scaled(synth.mag(), 0.01, "mag_small")
    st, og = gpu_store(cfg), oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    tr.load_inputs(torch.from_numpy(synth.nc_seeds(cfg, 0)).cuda())
    tr.capture(step0=0)                       # capture runs nothing; replays run the steps
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    opt = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    labels = synth.labels(cfg)
    for step in range(3):
        seeds = synth.nc_seeds(cfg, step)
        tr.load_inputs(torch.from_numpy(seeds).cuda())
        for k in synth.param_order(cfg):   # re-sync from the oracle state (see test_nc_step_parity)
            tr.pview(k).copy_(torch.from_numpy(params[k].astype(np.float32)))
            tr.pview(k, "m").copy_(torch.from_numpy(opt[k]["m"].astype(np.float32)))
            tr.pview(k, "v").copy_(torch.from_numpy(opt[k]["v"].astype(np.float32)))
        tr.replay()
        torch.cuda.synchronize()
        assert int(tr.counters[0].item()) == step + 1 and int(tr.counters[1].item()) == step + 1
        res = oracle.nc_step(og, params, seeds, labels, step, cfg.rng_seed)
        _compare_blocks(cfg, st, tr.sampler, res.blocks)
        close(tr.loss.cpu().numpy()[0], res.loss, what=f"graph step {step} loss")
        check_grads(tr, res, cfg, step)
        for k in synth.param_order(cfg):
            oracle.adam(params[k], res.grads[k], opt[k]["m"], opt[k]["v"], cfg.lr, step + 1)


@pytest.mark.parametrize("use_graph,fuse", [(True, True), (True, False), (False, True)])
def test_pipelined_steps_match_oracle(torch_cuda, use_graph, fuse):
    """Double-buffered pipeline (bench.py's default): batch k+1 is sampled on a side stream
    while batch k computes.  Every computed batch's blocks are bit-exact, its loss and grads
    match the oracle, and the device step / t counters advance as in the serial graph."""
    import torch
    cfg = synth.scaled(synth.mag(), 0.01, "mag_small")
    st, og = gpu_store(cfg), oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    tr.fuse_gather = fuse
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    opt = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    labels = synth.labels(cfg)
    dev_seeds = [torch.from_numpy(synth.nc_seeds(cfg, i)).cuda() for i in range(5)]
    tr.pipeline_start((dev_seeds[0],), 0, use_graph=use_graph)
    for step in range(4):
        for k in synth.param_order(cfg):   # re-sync from the oracle state (see test_nc_step_parity)
            tr.pview(k).copy_(torch.from_numpy(params[k].astype(np.float32)))
            tr.pview(k, "m").copy_(torch.from_numpy(opt[k]["m"].astype(np.float32)))
            tr.pview(k, "v").copy_(torch.from_numpy(opt[k]["v"].astype(np.float32)))
        tr.pipeline_step(dev_seeds[step + 1])
        tr.pipeline_sync()
        torch.cuda.synchronize()
        assert int(tr.counters[0].item()) == step + 2 and int(tr.counters[1].item()) == step + 1
        seeds = synth.nc_seeds(cfg, step)
        res = oracle.nc_step(og, params, seeds, labels, step, cfg.rng_seed)
        _compare_blocks(cfg, st, tr.sampler, res.blocks)
        close(tr.loss.cpu().numpy()[0], res.loss, what=f"pipelined step {step} loss")
        check_grads(tr, res, cfg, step)
        for k in synth.param_order(cfg):
            oracle.adam(params[k], res.grads[k], opt[k]["m"], opt[k]["v"], cfg.lr, step + 1)


@pytest.mark.parametrize("n,d,C", [(1024, 128, 349), (37, 128, 8), (300, 64, 153), (65, 32, 512), (129, 96, 33)])
def test_nc_loss_parity(torch_cuda, n, d, C):
    """gsb_nc_loss (tcgen05 logits / dh / dWc with split-K, softmax CE with the fused batch
    mean) against oracle.nc_loss at ragged shapes: loss, dh, dWc, dbc within 1e-5 (R-tol)."""
    import ctypes as C_
    import torch
    from paper_2406_06022_b200._lib import call
    rng = np.random.default_rng(n + d + C)
    h = rng.normal(size=(n, d)).astype(np.float32)
    Wc = (rng.normal(size=(d, C)) / np.sqrt(d)).astype(np.float32)
    bc = rng.normal(size=C).astype(np.float32) * 0.1
    y = rng.integers(0, C, size=n).astype(np.int32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ht, Wt, bt, yt = t(h), t(Wc), t(bc), t(y)
    gid = torch.arange(n, dtype=torch.int64, device="cuda")
    ldl = (C + 3) // 4 * 4
    logits = torch.zeros((n, ldl), dtype=torch.float32, device="cuda")
    rl = torch.zeros(n + 1024, dtype=torch.float32, device="cuda")
    loss = torch.zeros(1, dtype=torch.float32, device="cuda")
    dh = torch.zeros((n, d), dtype=torch.float32, device="cuda")
    dWc = torch.zeros((d, C), dtype=torch.float32, device="cuda")
    dbc = torch.zeros(C, dtype=torch.float32, device="cuda")
    P = lambda x: C_.c_void_p(x.data_ptr())
    for _ in range(2):      # the second call reuses the ticket word the first one reset
        call("gsb_nc_loss", P(ht), n, d, P(Wt), P(bt), C, P(yt), P(gid), 0, P(logits), P(rl), P(loss), P(dh), P(dWc),
             P(dbc), None)
    ol, _, odh, odW, odb = oracle.nc_loss(h, Wc, bc, y)
    close(loss.cpu().numpy()[0], ol, what="loss")
    close(dh.cpu().numpy(), odh, what="dh")
    close(dWc.cpu().numpy(), odW, what="dWc")
    close(dbc.cpu().numpy(), odb, what="dbc")
    # split form: gsb_nc_loss without dWc / dbc, then gsb_nc_loss_dw on a second stream that
    # waits for it (what the trainer does): the same kernels as the joined call
    dWc2 = torch.full((d, C), 7.0, dtype=torch.float32, device="cuda")
    dbc2 = torch.full((C,), 7.0, dtype=torch.float32, device="cuda")
    side = torch.cuda.Stream()
    call("gsb_nc_loss", P(ht), n, d, P(Wt), P(bt), C, P(yt), P(gid), 0, P(logits), P(rl), P(loss), P(dh), None, None,
         None)
    side.wait_stream(torch.cuda.current_stream())
    pad = torch.empty(d * ldl, dtype=torch.float32, device="cuda")
    call("gsb_nc_loss_dw", P(ht), n, d, P(logits), C, P(dWc2), P(dbc2), P(pad), C_.c_void_p(side.cuda_stream))
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    close(dWc2.cpu().numpy(), odW, what="dWc (gsb_nc_loss_dw)")
    close(dbc2.cpu().numpy(), odb, what="dbc (gsb_nc_loss_dw)")


@pytest.mark.parametrize("name,batch", [("mag_small", 2600), ("mag_small", 3000), ("mag_small", 3200),
                                        ("tiny", 700), ("tiny", 1500)])
def test_nc_step_splitk_batches(torch_cuda, name, batch):
    """Regression: batch sizes whose top-layer GEMM splits K across CTAs
    (few output tiles) with a split count that does not divide the K panels, and ntypes with
    fewer slots than the widest one.  Activations, loss and gradients within rtol."""
    import torch
    cfg = CASES[name]()
    cfg.batch = batch
    st, og = gpu_store(cfg), oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    seeds = synth.nc_seeds(cfg, 1)
    tr.forward_backward(torch_cuda.from_numpy(seeds).cuda(), 1)
    res = oracle.nc_step(og, params, seeds, synth.labels(cfg), 1, cfg.rng_seed)
    for l in range(len(cfg.fanouts)):
        nd = len(res.blocks[l].dst_gid)
        close(tr.hout[l][:nd].cpu().numpy(), res.hs[l], what=f"batch {batch} h{l}")
    close(tr.loss.cpu().numpy()[0], res.loss, what="loss")
    check_grads(tr, res, cfg, 1)


def test_gcn_homogeneous_step_parity(torch_cuda):
    """Table 3's workload (§8(f) f4): a homogeneous graph (one ntype, one relation,
    average degree 100, 64-d features) and a GCN (the RGCN layer with R = 1, R-gcn), at 1/1000
    of the 1B-edge size: blocks bit-exact, activations / loss / gradients within rtol."""
    import torch
    cfg = synth.gcn_1b(0.001)
    assert cfg.num_ntypes == 1 and cfg.num_etypes == 1
    st, og = gpu_store(cfg), oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    for step in (0, 1):
        seeds = synth.nc_seeds(cfg, step)
        tr.forward_backward(torch_cuda.from_numpy(seeds).cuda(), step)
        res = oracle.nc_step(og, params, seeds, synth.labels(cfg), step, cfg.rng_seed)
        _compare_blocks(cfg, st, tr.sampler, res.blocks)
        for l in range(len(cfg.fanouts)):
            nd = len(res.blocks[l].dst_gid)
            close(tr.hout[l][:nd].cpu().numpy(), res.hs[l], what=f"gcn step {step} h{l}")
        close(tr.loss.cpu().numpy()[0], res.loss, what="gcn loss")
        check_grads(tr, res, cfg, step)


@pytest.mark.parametrize("knob,value,case", [("GSB_TCSR", "1", "mag_small"), ("GSB_NC", "fused", "mag_small"),
                                             ("GSB_AGG_HALF", "2", "mag_small_bf16"),
                                             ("GSB_AGG_HALF", "0", "mag_small_bf16")])
def test_optin_paths_parity(torch_cuda, knob, value, case, monkeypatch):
    """The opt-in / size-selected paths keep parity: GSB_TCSR=1 (by-source transposed CSR per
    block + the deterministic gather scatter of the hidden layer's input gradient, §8(a) a4),
    GSB_NC=fused (the fused SIMT decoder: logits, softmax-CE, dh, dWc, dbc), GSB_AGG_HALF=2 (the
    half-warp-per-row layer-0 aggregation that large batches take, forced at a small one) and
    GSB_AGG_HALF=0 (the warp-per-row kernel, which the default quarter-warp kernel replaces for
    256-B rows)."""
    import torch
    monkeypatch.setenv(knob, value)
    cfg = CASES[case]()
    st, og = gpu_store(cfg), oracle_graph(cfg)
    tr = _gpu_trainer(cfg, st)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    for step in (0, 2):
        seeds = synth.nc_seeds(cfg, step)
        tr.forward_backward(torch_cuda.from_numpy(seeds).cuda(), step)
        res = oracle.nc_step(og, params, seeds, synth.labels(cfg), step, cfg.rng_seed)
        close(tr.loss.cpu().numpy()[0], res.loss, what=f"{knob} loss")
        check_grads(tr, res, cfg, step)
        if knob == "GSB_TCSR":    # the scatter's output: layer 1's input gradient (its ReLU mask is
            z = res.zs[0]            # applied inside layer 0's weight-gradient GEMM, so mask it here);
            n0 = z.shape[0]          # ambiguous units (|z| ~ 0) left out (R-relutie)
            keep = np.abs(z) > 1e-5 * np.abs(z).max()
            exp = np.where(z > 0, res.extra["dh"][0], 0.0)
            got = np.where(z > 0, tr.dh[0][:n0].cpu().numpy(), 0.0)
            close(got[keep], exp[keep], what="dh0 via the transposed CSR")
