"""GPU parity of Eq. 1 feature construction against the
oracle: fp32 and bf16 feature rows, 64-d and 768-d widths, ragged row ranges."""
import numpy as np
import pytest

import oracle
import synth
from tests._pair import close, gpu_store, oracle_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2406_06022_b200 import build
    build.build()
    return torch


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_construct_features_tiny(torch_cuda, dtype):
    cfg = synth.with_dtype(synth.tiny(), dtype)
    st, og = gpu_store(cfg), oracle_graph(cfg)
    # ntype 1 (B) receives r1 from A; ntype 0 (A) receives r0 from A and r3 from C
    for ntype, featured, first, count in [(1, [0], 0, cfg.counts[1]), (0, [0, 2], 17, 1001), (0, [2], 0, 333)]:
        got = st.construct_features(ntype, featured, cfg.feat_dim, first, count).cpu().numpy()
        exp = oracle.construct_features(og, ntype, featured, first=first, count=count)
        close(got, exp, what=f"F' ntype {ntype} from {featured}")


def test_construct_features_wide_bf16(torch_cuda):
    """MAG240M-shaped widths: authors built from their papers' 768-d bf16 rows."""
    cfg = synth.scaled(synth.mag240m(), 1.0 / 20000, "mag240m_tiny")
    st, og = gpu_store(cfg), oracle_graph(cfg)
    paper = cfg.ntypes.index("paper")
    author = cfg.ntypes.index("author")
    d = cfg.dim_of(paper)
    got = st.construct_features(author, [paper], d, 5, 700).cpu().numpy()
    exp = oracle.construct_features(og, author, [paper], first=5, count=700)
    close(got, exp, what="F' author from papers")
    assert np.abs(exp).sum() > 0


@pytest.mark.parametrize("dtype,dim", [("f32", 64), ("bf16", 768), ("bf16", 128)])
def test_construct_features_hubs(torch_cuda, dtype, dim):
    """Hub in-degrees around the head/tail split (featcon.cu kFeatconCap = 128): segments of
    0, 1, 127, 128, 129, 255, 256, 257, 1000 and 40 000 edges over two featured relations, in
    a range that starts and ends mid-graph.  Expected rows: the mean of the in-neighbours'
    rows (Eq. 1), written out in float64 from the COO."""
    torch = torch_cuda
    rng = np.random.default_rng(2406)
    nA, nB = 5000, 64
    degs = [0, 1, 127, 128, 129, 255, 256, 257, 1000, 40000, 3, 0, 129, 2]
    src, dst = [], []
    for r in range(2):
        s_r, d_r = [], []
        for v in range(nB):
            k = degs[(v + 5 * r) % len(degs)] if v % 3 else int(rng.integers(0, 6))
            s_r.append(rng.integers(0, nA, size=k))
            d_r.append(np.full(k, v))
        src.append(np.concatenate(s_r).astype(np.int32))
        dst.append(np.concatenate(d_r).astype(np.int32))
    from paper_2406_06022_b200.runtime import GraphStore
    st = GraphStore([nA, nB], [0, 0], [1, 1], "cuda")
    for r in range(2):
        st.load_etype(r, torch.from_numpy(src[r]), torch.from_numpy(dst[r]))
    F = rng.uniform(-1, 1, size=(nA, dim)).astype(np.float32)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    Ft = torch.from_numpy(F).to(tdt)
    st.set_features(0, Ft)
    st.set_features(1, torch.zeros((nB, dim), dtype=tdt))
    Fx = Ft.float().numpy().astype(np.float64)      # the stored (rounded) rows
    first, count = 3, nB - 7
    got = st.construct_features(1, [0], dim, first, count).cpu().numpy()
    s_all, d_all = np.concatenate(src), np.concatenate(dst)
    exp = np.zeros((count, dim))
    for i in range(count):
        nb = s_all[d_all == first + i]
        if nb.size:
            exp[i] = Fx[nb].mean(axis=0)
    close(got, exp, what=f"F' hubs {dtype} {dim}")
