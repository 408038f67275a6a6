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
