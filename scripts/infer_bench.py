"""Time full-graph layer-wise inference on the ogbn-mag-shaped graph (bf16
features): both RGCN layers over every node's whole neighbourhood, in chunks of consecutive
gids.  One JSON line: nodes/s per full inference and algorithmic GB/s of the aggregation
(per edge one source row + its 12-B index; per node the Acat row written, the self row read)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from bench import build_gsb  # noqa: E402
from paper_2406_06022_b200.runtime import FullGraphInference  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mag"
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 18
cfg = synth.with_dtype(synth.get(name), "bf16")
st, _ = build_gsb(cfg, torch.device("cuda"))
inf = FullGraphInference(st, synth.init_params(cfg), len(cfg.fanouts), cfg.hidden, chunk=chunk)
inf.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 3
for _ in range(reps):
    inf.run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
N, E = cfg.num_nodes, sum(int(x) for x in st.n_edges)
S = max(len([r for r in range(cfg.num_etypes) if cfg.etypes[r].dst == t]) for t in range(cfg.num_ntypes))
l0 = E * (cfg.feat_dim * 2 + 12) + N * (cfg.feat_dim * 2 + (S + 1) * cfg.feat_dim * 4)
l1 = E * (cfg.hidden * 4 + 12) + N * (cfg.hidden * 4 + (S + 1) * cfg.hidden * 4)
print(json.dumps({"what": f"full-graph inference, {name}-shaped (bf16 features), {len(cfg.fanouts)} RGCN layers, "
                          f"chunk {inf.chunk}", "nodes": N, "edges": E, "ms": ms, "nodes_per_s": N / ms * 1e3,
                  "agg_alg_GB": (l0 + l1) / 1e9, "agg_alg_GBps_over_whole_run": (l0 + l1) / ms / 1e6}))

# per-kernel breakdown of one more run (events around every launch; serialised)
import ctypes as C  # noqa: E402
from paper_2406_06022_b200 import _lib  # noqa: E402
_lib.lib().gsb_profile_enable(1)
inf.run()
torch.cuda.synchronize()
_lib.lib().gsb_profile_enable(0)
buf = C.create_string_buffer(1 << 16)
_lib.call("gsb_profile_dump", buf, len(buf))
rows = []
for line in buf.value.decode().splitlines():
    n, c, t = line.split()
    rows.append((float(t), n, int(c)))
rows.sort(reverse=True)
print(json.dumps({"profile_ms": {n: round(t, 3) for t, n, c in rows[:12]},
                  "launches": {n: c for t, n, c in rows[:12]}}))
