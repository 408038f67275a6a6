"""GPU parity of the negative samplers and score / loss variants of App. A (SURVEY §8(f)
f2): uniform negatives bit-exact, gsb_lp_score_ex (sampled / in-batch negatives, DistMult /
dot product, contrastive / CE / weighted CE) within rtol 1e-5, and the LP train step with
every sampler against the oracle."""
import ctypes as C

import zlib

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


def test_uniform_negatives_bitexact(torch_cuda):
    import torch
    from paper_2406_06022_b200._lib import call
    for (n_pos, K, n_nodes, base, step, pb) in [(4096, 32, 1_250_000, 7, 3, 0), (5, 2, 17, 0, 0, 11),
                                               (1000, 7, 99, 100, 12345, 3)]:
        out = torch.empty(n_pos * K, dtype=torch.int64, device="cuda")
        call("gsb_uniform_negatives", n_pos, K, n_nodes, base, 77, step, None, pb, C.c_void_p(out.data_ptr()), None)
        exp = oracle.uniform_negatives(n_pos, K, n_nodes, base, 77, step, pb)
        assert np.array_equal(out.cpu().numpy(), exp)


SCORE_CASES = [(s, sc, k, 96) for s in ("joint", "uniform", "in_batch") for sc in ("distmult", "dot") for k in (0, 1, 2)]
# in-batch with B % 32 != 0 takes the SIMT kernel instead of the tensor-core contractions
SCORE_CASES += [("in_batch", "distmult", 0, 50), ("in_batch", "dot", 2, 50), ("in_batch", "distmult", 1, 512)]


@pytest.mark.parametrize("sampler,score,kind,B", SCORE_CASES)
def test_lp_score_ex_parity(torch_cuda, sampler, score, kind, B):
    import torch
    from paper_2406_06022_b200._lib import call
    rng = np.random.default_rng(zlib.crc32(f"{sampler}/{score}/{kind}/{B}".encode()))
    d, n_rows = 128, 2 * B + 50
    K = B - 1 if sampler == "in_batch" else 8
    mode = 1 if sampler == "in_batch" else 0
    group = 1 if sampler == "uniform" else K
    n_neg = 0 if mode else (B * K if sampler == "uniform" else -(-B // K) * K)
    H = rng.standard_normal((n_rows, d)).astype(np.float32)
    rel = rng.standard_normal(d).astype(np.float32)
    w = rng.uniform(0.25, 2.0, B).astype(np.float32)
    iu, iv = rng.integers(0, n_rows, B).astype(np.int32), rng.integers(0, n_rows, B).astype(np.int32)
    ineg = rng.integers(0, n_rows, max(n_neg, 1)).astype(np.int32)
    T = lambda a: torch.from_numpy(a).cuda()
    P = lambda x: C.c_void_p(x.data_ptr()) if x is not None else None
    Hd, reld, wd, iud, ivd, inegd = T(H), T(rel), T(w), T(iu), T(iv), T(ineg)
    scores = torch.empty((B, K + 1), device="cuda")
    rl = torch.empty(B, device="cuda")
    loss = torch.empty(1, device="cuda")
    dH = torch.empty_like(Hd)
    drel = torch.zeros_like(reld)
    dm = score == "distmult"
    wb = C.c_size_t()
    call("gsb_lp_score_ws_bytes", B, d, mode, C.byref(wb))
    ws = torch.empty(max(wb.value, 1), dtype=torch.uint8, device="cuda")
    call("gsb_lp_score_ex", P(Hd), n_rows, d, P(iud), P(ivd), P(inegd) if n_neg else None, B, K, group, mode,
         P(reld) if dm else None, kind, P(wd), P(scores), P(rl), P(loss), P(dH), P(drel) if dm else None, P(ws),
         ws.numel(), None)
    H64 = H.astype(np.float64)
    l, sc, dhu, dhv, dhn, dr = oracle.lp_loss_ex(H64[iu], H64[iv], H64[ineg[:n_neg]] if n_neg else None,
                                                 rel.astype(np.float64) if dm else None, K, group, mode, kind,
                                                 w.astype(np.float64))
    close(scores.cpu().numpy(), sc, what="scores")
    close(loss.cpu().numpy()[0], l, what="loss")
    dHe = np.zeros((n_rows, d))
    np.add.at(dHe, iu, dhu)
    np.add.at(dHe, iv, dhv)
    if n_neg:
        np.add.at(dHe, ineg[:n_neg], dhn)
    close(dH.cpu().numpy(), dHe, what="dH")
    if dm:
        close(drel.cpu().numpy(), dr, what="drel")


def test_lp_score_ex_rejects_bad_layouts(torch_cuda):
    import torch
    from paper_2406_06022_b200._lib import GsbError, call
    x = torch.zeros(64 * 8, device="cuda")
    p = C.c_void_p(x.data_ptr())
    with pytest.raises(GsbError):      # in-batch needs K = B - 1
        call("gsb_lp_score_ex", p, 8, 8, p, p, None, 8, 3, 1, 1, None, 0, None, p, p, p, p, None, None, 0, None)
    with pytest.raises(GsbError):      # weighted CE needs weights
        call("gsb_lp_score_ex", p, 8, 8, p, p, p, 8, 2, 2, 0, None, 2, None, p, p, p, p, None, None, 0, None)
    with pytest.raises(GsbError):      # in-batch on the tensor cores needs its workspace
        call("gsb_lp_score_ex", p, 8, 8, p, p, None, 64, 63, 1, 1, None, 0, None, p, p, p, p, None, None, 0, None)


def _keep(cfg):
    k = synth.lp_keep_mask(cfg).astype(np.uint8)
    keep = {cfg.lp_etype: k}
    if cfg.lp_rev_etype >= 0:
        keep[cfg.lp_rev_etype] = k
    return keep


@pytest.fixture(scope="module")
def lp_tiny(torch_cuda):
    cfg = synth.tiny_lp()
    keep = _keep(cfg)
    return cfg, gpu_store(cfg, keep=keep), oracle_graph(cfg, keep=keep)


@pytest.mark.parametrize("sampler,score,kind", [("uniform", "distmult", 0), ("local_joint", "distmult", 0),
                                                ("in_batch", "distmult", 0), ("joint", "dot", 1),
                                                ("uniform", "dot", 2)])
def test_lp_step_samplers_parity(lp_tiny, torch_cuda, sampler, score, kind):
    """One LP step per sampler / score / loss: negatives and seed set bit-exact, scores, loss
    and gradients within rtol (R-tol, R-relutie)."""
    import torch
    from paper_2406_06022_b200.runtime import LPTrainer
    cfg, st, og = lp_tiny
    dst_t = cfg.etypes[cfg.lp_etype].dst
    local = (cfg.counts[dst_t] // 4, cfg.counts[dst_t] // 2) if sampler == "local_joint" else None
    names = [k for k in synth.param_order(cfg) if score == "distmult" or k != "rel"]
    p32 = {k: v for k, v in synth.init_params(cfg).items() if k in names}
    tr = LPTrainer(st, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_neg, cfg.lp_etype, cfg.lp_rev_etype,
                   p32, names, lr=cfg.lr, rng_seed=cfg.rng_seed, loss_kind=kind, neg_sampler=sampler, score=score,
                   local_range=local)
    w = np.random.default_rng(5).uniform(0.5, 1.5, cfg.batch)
    tr.pos_w.copy_(torch.from_numpy(w.astype(np.float32)))
    params = {k: v.astype(np.float64) for k, v in p32.items()}
    step = 1
    u, v = synth.lp_train_edges(cfg, step)
    dev = lambda a: torch.from_numpy(np.asarray(a, np.int64)).cuda()
    tr.forward_backward(dev(u), dev(v), step)
    res = oracle.lp_step(og, params, u, v, step, cfg.rng_seed, loss_kind=kind, neg_sampler=sampler, score=score,
                         local_range=local, w=w.astype(np.float32).astype(np.float64))
    if tr.n_neg:
        assert np.array_equal(tr.neg[:tr.n_neg].cpu().numpy(), res.extra["neg"])
    ns = int(tr.n_seeds.item())
    assert np.array_equal(tr.seeds[:ns].cpu().numpy(), res.extra["seeds"])
    close(tr.scores.cpu().numpy(), res.extra["scores"], what="scores")
    close(tr.loss.cpu().numpy()[0], res.loss, what="loss")
    L = len(cfg.fanouts)
    slack = {}
    for l in range(L - 1):
        sW, sb, _ = relu_tie_slack(res, cfg.num_etypes, l)
        slack[f"W{l}"], slack[f"b{l}"] = sW, sb
    for k in names:
        g = tr.pview(k, "g").cpu().numpy()
        if k in slack:
            close_slack(g, res.grads[k], slack[k], what=f"grad {k}")
        else:
            close(g, res.grads[k], what=f"grad {k}")
