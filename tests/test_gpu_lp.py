"""GPU parity of the link-prediction path (§8(a) a3', a9, a10): joint negatives and LP seed
set bit-exact, target-edge exclusion inside sampling bit-exact, DistMult + contrastive / CE
loss and gradients within rtol 1e-5, and the whole LP train step."""
import ctypes as C

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


def _keep(cfg):
    k = synth.lp_keep_mask(cfg).astype(np.uint8)
    keep = {cfg.lp_etype: k}
    if cfg.lp_rev_etype >= 0:
        keep[cfg.lp_rev_etype] = k
    return keep


CASES = {"tiny_lp": lambda: synth.tiny_lp(),
         "amazon_small": lambda: synth.scaled(synth.amazon_lp(), 1.0 / 400, "amazon_small")}


@pytest.fixture(scope="module", params=list(CASES))
def lp_pair(request, torch_cuda):
    cfg = CASES[request.param]()
    keep = _keep(cfg)
    return cfg, gpu_store(cfg, keep=keep), oracle_graph(cfg, keep=keep)


def test_joint_negatives_bitexact(torch_cuda):
    import torch
    from paper_2406_06022_b200._lib import call
    for (n_pos, K, n_nodes, base, step, gb) in [(4096, 32, 1_250_000, 7, 3, 0), (5, 2, 17, 0, 0, 11),
                                               (1000, 7, 99, 100, 12345, 3)]:
        G = (n_pos + K - 1) // K
        out = torch.empty(G * K, dtype=torch.int64, device="cuda")
        call("gsb_joint_negatives", n_pos, K, n_nodes, base, 77, step, None, gb, C.c_void_p(out.data_ptr()), None)
        exp = oracle.joint_negatives(n_pos, K, n_nodes, base, 77, step, gb)
        assert np.array_equal(out.cpu().numpy(), exp)


def test_lp_seeds_bitexact(torch_cuda):
    import torch
    from paper_2406_06022_b200._lib import call
    rng = np.random.default_rng(1)
    B, n_neg = 300, 320
    u = rng.integers(0, 5000, B)
    v = rng.integers(0, 5000, B)
    neg = rng.integers(0, 5000, n_neg)
    t = lambda a: torch.from_numpy(np.asarray(a, np.int64)).cuda()
    seeds = torch.empty(2 * B + n_neg, dtype=torch.int64, device="cuda")
    ns = torch.zeros(1, dtype=torch.int64, device="cuda")
    iu, iv = (torch.empty(B, dtype=torch.int32, device="cuda") for _ in range(2))
    ineg = torch.empty(n_neg, dtype=torch.int32, device="cuda")
    wb = C.c_size_t()
    call("gsb_lp_seeds_bytes", B, n_neg, C.byref(wb))
    ws = torch.empty(wb.value, dtype=torch.uint8, device="cuda")
    U, V, N = t(u), t(v), t(neg)
    P = lambda x: C.c_void_p(x.data_ptr())
    call("gsb_lp_seeds", P(U), P(V), B, P(N), n_neg, P(seeds), P(ns), P(iu), P(iv), P(ineg), P(ws), ws.numel(), None)
    exp = oracle.lp_seeds(u, v, neg)
    n = int(ns.item())
    assert n == len(exp) and np.array_equal(seeds[:n].cpu().numpy(), exp)
    assert np.array_equal(iu.cpu().numpy(), np.searchsorted(exp, u))
    assert np.array_equal(iv.cpu().numpy(), np.searchsorted(exp, v))
    assert np.array_equal(ineg.cpu().numpy(), np.searchsorted(exp, neg))


def test_sample_with_exclusion_bitexact(lp_pair, torch_cuda):
    from paper_2406_06022_b200.runtime import MiniBatchSampler
    from tests.test_gpu_parity import _compare_blocks
    cfg, st, og = lp_pair
    for step in (0, 2):
        u, v = synth.lp_train_edges(cfg, step)
        et = cfg.etypes[cfg.lp_etype]
        neg = oracle.joint_negatives(len(u), cfg.num_neg, cfg.counts[et.dst], int(cfg.node_off[et.dst]),
                                     cfg.rng_seed, step)
        seeds = oracle.lp_seeds(u, v, neg)
        sm = MiniBatchSampler(st, cfg.fanouts, max_seeds=len(seeds), max_excl=len(u))
        dev = lambda a: torch_cuda.from_numpy(np.asarray(a, np.int64)).cuda()
        sm.sample(dev(seeds), cfg.rng_seed, step, dev(u), dev(v), cfg.lp_etype, cfg.lp_rev_etype)
        assert sm.poll_error() == 0
        ob = oracle.sample_blocks(og, seeds, cfg.fanouts, cfg.rng_seed, step, u, v, cfg.lp_etype, cfg.lp_rev_etype)
        _compare_blocks(cfg, st, sm, ob)
        # exclusion soundness on the GPU blocks themselves
        for l in range(len(cfg.fanouts)):
            b = sm.block(l)
            pairs = set(zip(u.tolist(), v.tolist()))
            src = b.e_src_gid.cpu().numpy()
            seg = b.seg_ptr.cpu().numpy()
            dst = b.dst_gid.cpu().numpy()
            S = b.num_slots
            slots = st.slot_etypes()
            tdst = np.searchsorted(cfg.node_off, dst, side="right") - 1
            for j in range(len(dst)):
                for s, r in enumerate(slots[tdst[j]]):
                    e = slice(seg[j * S + s], seg[j * S + s + 1])
                    if r == cfg.lp_etype:
                        assert not any((int(x), int(dst[j])) in pairs for x in src[e])
                    if r == cfg.lp_rev_etype:
                        assert not any((int(dst[j]), int(x)) in pairs for x in src[e])


@pytest.mark.parametrize("kind", [0, 1])
def test_lp_score_parity(torch_cuda, kind):
    import torch
    from paper_2406_06022_b200._lib import call
    rng = np.random.default_rng(4 + kind)
    B, K, d, n_rows = 96, 8, 128, 150
    H = rng.standard_normal((n_rows, d)).astype(np.float32)
    rel = rng.standard_normal(d).astype(np.float32)
    iu, iv = rng.integers(0, n_rows, B).astype(np.int32), rng.integers(0, n_rows, B).astype(np.int32)
    ineg = rng.integers(0, n_rows, (B // K) * K).astype(np.int32)
    T = lambda a: torch.from_numpy(a).cuda()
    P = lambda x: C.c_void_p(x.data_ptr())
    Hd, reld, iud, ivd, inegd = T(H), T(rel), T(iu), T(iv), T(ineg)
    scores = torch.empty((B, K + 1), device="cuda")
    rl = torch.empty(B, device="cuda")
    loss = torch.empty(1, device="cuda")
    dH = torch.empty_like(Hd)
    drel = torch.empty_like(reld)
    call("gsb_lp_score", P(Hd), n_rows, d, P(iud), P(ivd), P(inegd), B, K, P(reld), kind, P(scores), P(rl),
         P(loss), P(dH), P(drel), None)
    H64 = H.astype(np.float64)
    l, sc, dhu, dhv, dhn, dr = oracle.lp_loss(H64[iu], H64[iv], H64[ineg], rel.astype(np.float64), K, kind)
    close(scores.cpu().numpy(), sc, what="scores")
    close(loss.cpu().numpy()[0], l, what="loss")
    dHe = np.zeros((n_rows, d))
    np.add.at(dHe, iu, dhu)
    np.add.at(dHe, iv, dhv)
    np.add.at(dHe, ineg, dhn)
    close(dH.cpu().numpy(), dHe, what="dH")
    close(drel.cpu().numpy(), dr, what="drel")


def test_lp_step_parity(lp_pair, torch_cuda):
    import torch
    from paper_2406_06022_b200.runtime import LPTrainer
    from tests.test_gpu_parity import _adam_interval, check_grads
    cfg, st, og = lp_pair
    tr = LPTrainer(st, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_neg, cfg.lp_etype, cfg.lp_rev_etype,
                   synth.init_params(cfg), synth.param_order(cfg), lr=cfg.lr, rng_seed=cfg.rng_seed)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    opt = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    rtol = 1e-5
    for step in range(2):
        for k in synth.param_order(cfg):
            tr.pview(k).copy_(torch.from_numpy(params[k].astype(np.float32)))
            tr.pview(k, "m").copy_(torch.from_numpy(opt[k]["m"].astype(np.float32)))
            tr.pview(k, "v").copy_(torch.from_numpy(opt[k]["v"].astype(np.float32)))
        tr.t = step
        u, v = synth.lp_train_edges(cfg, step)
        dev = lambda a: torch.from_numpy(np.asarray(a, np.int64)).cuda()
        tr.forward_backward(dev(u), dev(v), step)
        res = oracle.lp_step(og, params, u, v, step, cfg.rng_seed)
        assert np.array_equal(tr.neg.cpu().numpy(), res.extra["neg"])
        ns = int(tr.n_seeds.item())
        assert np.array_equal(tr.seeds[:ns].cpu().numpy(), res.extra["seeds"])
        close(tr.scores.cpu().numpy(), res.extra["scores"], what=f"step {step} scores")
        close(tr.loss.cpu().numpy()[0], res.loss, what="loss")
        # MRR of this step's scores: the same fp32 scores on both sides (R-mrr)
        rr_o, mrr_o = oracle.lp_mrr(tr.scores.cpu().numpy())
        close(tr.mrr().cpu().numpy()[0], mrr_o, what="MRR")
        assert np.array_equal(np.rint(2 / tr.rr.cpu().numpy()), np.rint(2 / rr_o))
        slack = check_grads(tr, res, cfg, step)
        tr.optimizer_step()
        for k in synth.param_order(cfg):
            g = res.grads[k]
            tol_g = rtol * np.abs(g) + rtol * np.abs(g).max() + slack.get(k, 0.0)
            lo, hi, mid = _adam_interval(params[k], g, opt[k]["m"], opt[k]["v"], tol_g, cfg.lr, step + 1)
            gp = tr.pview(k).cpu().numpy().astype(np.float64)
            pslack = rtol * np.abs(mid) + rtol * np.abs(mid).max()
            assert not ((gp < lo - pslack) | (gp > hi + pslack)).any(), f"step {step} param {k}"
            oracle.adam(params[k], g, opt[k]["m"], opt[k]["v"], cfg.lr, step + 1)


def test_lp_pipelined_matches_oracle(lp_pair, torch_cuda):
    """LP through the double-buffered graph pipeline: negatives, seed set, loss and grads of
    every computed batch match the oracle (batch k+1's negatives/sampling run on the side
    stream during batch k's compute)."""
    import torch
    from paper_2406_06022_b200.runtime import LPTrainer
    from tests.test_gpu_parity import check_grads
    cfg, st, og = lp_pair
    tr = LPTrainer(st, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_neg, cfg.lp_etype, cfg.lp_rev_etype,
                   synth.init_params(cfg), synth.param_order(cfg), lr=cfg.lr, rng_seed=cfg.rng_seed)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    opt = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    dev = lambda a: torch.from_numpy(np.asarray(a, np.int64)).cuda()
    batches = [synth.lp_train_edges(cfg, i) for i in range(4)]
    tr.pipeline_start((dev(batches[0][0]), dev(batches[0][1])), 0)
    for step in range(3):
        for k in synth.param_order(cfg):
            tr.pview(k).copy_(torch.from_numpy(params[k].astype(np.float32)))
            tr.pview(k, "m").copy_(torch.from_numpy(opt[k]["m"].astype(np.float32)))
            tr.pview(k, "v").copy_(torch.from_numpy(opt[k]["v"].astype(np.float32)))
        tr.pipeline_step(dev(batches[step + 1][0]), dev(batches[step + 1][1]))
        tr.pipeline_sync()
        torch.cuda.synchronize()
        u, v = batches[step]
        res = oracle.lp_step(og, params, u, v, step, cfg.rng_seed)
        assert np.array_equal(tr.neg.cpu().numpy(), res.extra["neg"])
        ns = int(tr.n_seeds.item())
        assert np.array_equal(tr.seeds[:ns].cpu().numpy(), res.extra["seeds"])
        close(tr.loss.cpu().numpy()[0], res.loss, what=f"pipelined step {step} loss")
        check_grads(tr, res, cfg, step)
        for k in synth.param_order(cfg):
            oracle.adam(params[k], res.grads[k], opt[k]["m"], opt[k]["v"], cfg.lr, step + 1)


@pytest.mark.parametrize("B,K,ld", [(1, 1, 2), (1000, 32, 33), (77, 100, 104), (4096, 4095, 4096)])
def test_lp_mrr_parity(torch_cuda, B, K, ld):
    """gsb_lp_mrr vs oracle.lp_mrr (R-mrr) on scores with many exact ties (small integers)
    and ragged widths; ranks compared exactly (2 * rank is an integer), MRR within 1e-5."""
    import torch
    from paper_2406_06022_b200._lib import GsbError, call
    rng = np.random.default_rng(B + K)
    S = rng.integers(-3, 4, size=(B, ld)).astype(np.float32)
    S[: B // 2] += rng.normal(size=(B // 2, ld)).astype(np.float32)     # half the rows tie-free
    St = torch.from_numpy(S).cuda()
    rr = torch.empty(B, dtype=torch.float32, device="cuda")
    m = torch.empty(1, dtype=torch.float32, device="cuda")
    call("gsb_lp_mrr", C.c_void_p(St.data_ptr()), ld, B, K, C.c_void_p(rr.data_ptr()), C.c_void_p(m.data_ptr()), None)
    rr_o, m_o = oracle.lp_mrr(S[:, : K + 1])
    assert np.array_equal(np.rint(2 / rr.cpu().numpy()), np.rint(2 / rr_o))
    close(m.cpu().numpy()[0], m_o, what="MRR")
    with pytest.raises(GsbError):
        call("gsb_lp_mrr", C.c_void_p(St.data_ptr()), K, B, K, C.c_void_p(rr.data_ptr()), C.c_void_p(m.data_ptr()),
             None)
