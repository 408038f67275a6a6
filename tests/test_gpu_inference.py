"""GPU parity of full-graph layer-wise inference against the oracle: every
node's h_l over its whole neighbourhood, in ragged chunks, fp32 and bf16 features, and the
decoder's predictions / accuracy (argmax decisions compared where the oracle's top-2 margin
exceeds the tolerance)."""
import numpy as np
import pytest

import oracle
import synth
from tests._pair import RTOL_F32, close, gpu_store, oracle_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2406_06022_b200 import build
    build.build()
    return torch


@pytest.mark.parametrize("dtype,chunk", [("f32", 3000), ("bf16", 4096), ("f32", 1 << 20)])
def test_full_graph_inference(torch_cuda, dtype, chunk):
    import torch
    from paper_2406_06022_b200.runtime import FullGraphInference
    cfg = synth.with_dtype(synth.tiny(), dtype)
    st, og = gpu_store(cfg), oracle_graph(cfg)
    p32 = synth.init_params(cfg)
    params = {k: v.astype(np.float64) for k, v in p32.items()}
    inf = FullGraphInference(st, p32, len(cfg.fanouts), cfg.hidden, chunk=chunk)
    inf.run()
    torch.cuda.synchronize()
    hs = oracle.full_graph_infer(og, params)
    for l in range(len(cfg.fanouts)):
        close(inf.H[l].cpu().numpy(), hs[l], what=f"h{l} (all nodes)")
    t = cfg.target_ntype
    gids = np.arange(cfg.counts[t], dtype=np.int64) + cfg.node_off[t]
    labels = synth.labels(cfg)
    pred, correct = inf.predict(torch.from_numpy(gids).cuda(), torch.from_numpy(labels), int(cfg.node_off[t]),
                                cfg.num_classes)
    _, opred, margin = oracle.nc_predict(hs[-1][gids], params["Wc"], params["bc"])
    logit_scale = np.abs(hs[-1][gids] @ params["Wc"]).max()
    sure = margin > 4 * RTOL_F32 * logit_scale
    assert sure.mean() > 0.9
    assert np.array_equal(pred.cpu().numpy()[sure], opred[sure])
    ocorrect = int((opred == labels).sum())
    assert abs(correct - ocorrect) <= int((~sure).sum())
