#!/usr/bin/env python
"""bench.py -- RGCN mini-batch train step on B200 (GraphStorm arXiv 2406.06022 hot path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gsb|reference] [--config mag]

One step = one pass of the whole hot path over one mini-batch of synthetic input
(SURVEY.md §8(a)): seed batch -> per-etype fanout sampling (2 hops) -> relabel -> feature
gather -> 2 RGCN layers -> NC decoder + softmax CE -> backward -> (N>1: NCCL gradient
all-reduce) -> Adam.  Rank 0 prints ONE JSON line.  `--impl reference` times the CPU
oracle (the only other place bench.py executes oracle/) on bounded samples.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "RGCN train seeds/sec (and sampled edges/sec) on B200"
UNIT = "seeds/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="gsb", choices=["gsb", "reference"])
    ap.add_argument("--config", default="mag", choices=["mag", "tiny", "synth_1b", "synth_10b", "gcn_1b", "amazon_lp",
                                                        "tiny_lp", "mag240m", "mag240m_1_16"])
    ap.add_argument("--feat-dtype", default="auto", choices=["auto", "f32", "bf16"],
                    help="feature storage type; compute stays fp32 (auto: bf16 for the large configs, as "
                         "SURVEY §8(d) plans, fp32 for tiny)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--neg", default="joint", choices=["joint", "uniform", "local_joint", "in_batch"],
                    help="LP negative sampler (App. A.2.1)")
    ap.add_argument("--learnable-emb", action="store_true",
                    help="featureless ntypes (encoder configs) get learnable tables + sparse Adagrad (§8(f) f1)")
    ap.add_argument("--score", default="distmult", choices=["distmult", "dot"], help="LP score function (App. A.1)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="bounded oracle sample (cpu_baseline)")
    ap.add_argument("--profile-steps", type=int, default=20)
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--pipeline", default="on", choices=["on", "off"],
                    help="sample batch i+1 on a side stream while batch i computes (double-buffered)")
    ap.add_argument("--peer-gather", default="unique", choices=["unique", "fused"],
                    help="peer mode: gather the unique input rows over NVLink first (unique) or read them per "
                         "edge inside the fused aggregation (fused)")
    ap.add_argument("--topology", default="partitioned", choices=["partitioned", "replicate"],
                    help="N>1 graph store: CSC partitioned by dst node ID, remote segments read over NVLink by "
                         "the sampling kernels (partitioned, default; §8(e)), or the whole CSC on every rank")
    ap.add_argument("--sampling", default="peer", choices=["peer", "nccl"],
                    help="partitioned topology: read remote CSC segments over NVLink inside the sampling kernels "
                         "(peer), or send the frontier to its owners and the sampled edges back with NCCL "
                         "all-to-alls (nccl: §8(e) C2/C3, owner-side sampling; implies --features alltoall, eager steps)")
    ap.add_argument("--features", default="peer", choices=["peer", "alltoall", "replicate"],
                    help="N>1 feature store: partitioned by node ID and read over NVLink inside the kernels "
                         "(peer, default), partitioned + NCCL all-to-all fetch (alltoall), or replicated")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def config_for(name: str) -> synth.Config:
    return synth.get(name)


LP_OPTS = {"neg": "joint", "score": "distmult", "learnable_emb": False}


def lp_task(cfg: synth.Config) -> str:
    neg = LP_OPTS["neg"]
    negs = "in-batch" if neg == "in_batch" else f"{neg.replace('_', '-')}-{cfg.num_neg}"
    score = "DistMult" if LP_OPTS["score"] == "distmult" else "dot-product"
    return f"RGCN + {score} LP train step ({negs} negatives, contrastive)"


def cfg_json(cfg: synth.Config, n_gpus: int, extra=None) -> dict:
    task = "RGCN NC train step" if cfg.task == "nc" else lp_task(cfg)
    d = {"workload": f"{cfg.name}-shaped synthetic heterograph, {task}",
         "ntypes": cfg.num_ntypes, "etypes": cfg.num_etypes, "nodes": cfg.num_nodes, "edges": cfg.num_edges,
         "feat_dim": cfg.feat_dim, "fanouts": cfg.fanouts, "batch_per_gpu": cfg.batch,
         "global_batch": cfg.batch * n_gpus, "hidden": cfg.hidden, "num_classes": cfg.num_classes,
         "layers": len(cfg.fanouts), "optimizer": "adam",
         "parallelism": "single" if n_gpus == 1 else f"dp{n_gpus} (graph replicated, NCCL grad all-reduce)",
         "l2": "inputs larger than L2: feature table + CSC >> 126 MB, fresh random seed batch every step"}
    if getattr(cfg, "feat_dims", None):
        d["feat_dims"] = list(cfg.feat_dims)        # per ntype stored width (input encoder where projected)
        d["projected"] = [bool(x) for x in cfg.project]
    if LP_OPTS["learnable_emb"] and any(getattr(cfg, "project", None) or []):
        d["featureless_inputs"] = "learnable tables, sparse Adagrad on touched rows"
    if extra:
        d.update(extra)
    return d


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock + throttle reasons through NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.02):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------ roofline
def peaks():
    p = {"hbm_gbs": None, "src": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(path))
        p = {"hbm_gbs": float(j["hbm_gbs"]), "bf16_tflops": float(j.get("bf16_tflops", 0)),
             "bf16_tflops_sustained": float(j.get("bf16_tflops_sustained", 0)),
             "sm_max_mhz": float(j.get("sm_max_mhz", 1965.0)), "src": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0,
             "src": "fallback (B200_PROFILING.md)"}
    # FP32 FFMA peak: 148 SMs x 128 FP32 lanes x 2 flop x max SM clock
    p["fp32_tflops"] = 148 * 128 * 2 * p.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    return p


def kernel_work(name: str, sz: dict, cfg: synth.Config):
    """Algorithmic bytes (HBM-bound kernels) or flops (GEMMs) of `name` over ONE STEP with block
    sizes sz: SURVEY §8(d)'s per-unit figures x the units of the step.
      gather / aggregation: per sampled edge one d-wide source row + a 4-B index; per dst row its
        self row; per non-empty (dst, relation) segment one fp32 mean row written (the copy of
        the self row into the GEMM operand is not counted);
      sampling fill: per (dst, relation) 16 B of indptr; per sampled edge 4 B index read + 16 B
        (src gid, eid) written;
      GEMMs: 2 M N K flop (the 3xTF32 split is not counted)."""
    d0, hd, C = cfg.feat_dim, cfg.hidden, cfg.num_classes
    lay = None
    if name[-3:-1] == "_l" and name[-1].isdigit():
        lay = int(name[-1])
        name = name[:-3]
    fe = 2 if cfg.feat_dtype == "bf16" else 4      # feature element bytes (layer-0 inputs)
    if name == "gather":
        n = sz["n_src"][0]
        return "bytes", n * d0 * fe * 2 + n * 4
    if name == "rgcn_agg" and lay is not None:
        d = d0 if lay == 0 else hd
        es = fe if lay == 0 else 4
        return "bytes", (sz["n_edges"][lay] * (d * es + 4) + sz["n_dst"][lay] * d * es +
                         sz["nonempty_segs"][lay] * d * 4)
    if name == "sample_fill":
        return "bytes", sum(16 * sz["dst_rel"][l] + 20 * sz["n_edges"][l] for l in range(len(cfg.fanouts)))
    if name in ("rgcn_gemm_fwd", "rgcn_gemm_dW", "rgcn_gemm_dA") and lay is not None:
        return "flops", 2 * sz["acat_cols"][lay] * hd
    if name in ("enc_gemm_fwd", "enc_gemm_dW") and cfg.has_encoder:
        # a6: HBM bytes of the gathered bf16 rows of projected ntypes (+ the fp32 H0 rows written
        # by the forward / the split dH0 rows read by the backward)
        rows = sum(sz["src_type_cnt0"][t] for t in range(cfg.num_ntypes) if cfg.project[t])
        dims = max(cfg.dim_of(t) for t in range(cfg.num_ntypes) if cfg.project[t])
        return "bytes", rows * dims * 2 + rows * cfg.feat_dim * 4
    if name in ("nc_logits", "nc_gemm_dWc", "nc_gemm_dh"):
        return "flops", 2 * cfg.batch * hd * C
    return None, None


def traffic_of(cfg, name):
    """DRAM bytes per launch of `name` from the ncu --set full capture recorded in
    profiles/roofline_traffic.json for this config (dram__bytes_read.sum + write.sum)."""
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
        e = tj.get(f"{cfg.name}:{name}")
        return (e["bytes"], e["capture"]) if e else (None, None)
    except Exception:
        return None, None


def roofline_of(name, prof, sizes, cfg, pk, profile_steps):
    """Roofline entry of kernel `name`: algorithmic work per launch (kernel_work per step /
    launches per step) / its mean CUDA-event launch time, against the measured peak; DRAM
    traffic per launch from the ncu capture (profiles/roofline_traffic.json) and the DRAM
    fraction it implies at the same launch time."""
    kind, _ = kernel_work(name, sizes[0], cfg)
    if kind is None or name not in prof:
        return None
    lps = prof[name]["launches"] / profile_steps
    per_launch_work = float(np.mean([kernel_work(name, s, cfg)[1] for s in sizes])) / lps
    avg_ms = prof[name]["total_ms"] / prof[name]["launches"]
    if kind == "bytes":
        ach = per_launch_work / (avg_ms / 1e3) / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": ach / pk["hbm_gbs"], "traffic": None, "peak_src": pk["src"]}
    else:
        # tcgen05 kind::tf32 (3xTF32: 3 MMAs per fp32 product; achieved counts the algorithmic
        # 2*M*N*K once) against the dense TF32 peak = measured bf16 burst x 1/2 (guide ratio)
        ach = per_launch_work / (avg_ms / 1e3) / 1e12
        tf32 = pk.get("bf16_tflops", 1590.0) * 0.5
        roof = {"kernel": name, "bound": "tensor", "achieved": ach, "peak": tf32, "unit": "TFLOP/s",
                "frac": ach / tf32, "traffic": None,
                "peak_src": "dense TF32 = measured bf16 burst (MEASURED_PEAKS.json) x 0.5 (nominal ratio)"}
    tb, tsrc = traffic_of(cfg, name)
    if tb is not None:
        roof["traffic"] = tb
        roof["traffic_src"] = tsrc
        roof["dram_frac"] = tb / (avg_ms / 1e3) / 1e9 / pk["hbm_gbs"]
    roof["avg_launch_us"] = avg_ms * 1e3
    roof["launches_per_step"] = lps
    roof["algorithmic_per_launch"] = per_launch_work
    return roof


# ------------------------------------------------------------------------------ gsb arm
def build_gsb(cfg, device, partition=None, mode="peer", topology="replicate", sampling="peer"):
    """partition = (world, rank) -> features partitioned by node ID: mode "peer" maps every
    rank's shard over NVLink (PeerFeatures), "alltoall" fetches rows with NCCL (FeatureExchange).
    topology "partitioned" (with a partition): every rank builds only the CSC of the dst nodes
    it owns and maps the others' shards over NVLink (PeerCSC)."""
    import torch
    from paper_2406_06022_b200.runtime import GraphStore, LPTrainer, RGCNTrainer
    st = GraphStore(cfg.counts, cfg.etype_src(), cfg.etype_dst(), device)
    keep = None
    if cfg.task == "lp":   # val/test edges of the target etype (and its reverse) leave the graph
        k = torch.from_numpy(synth.lp_keep_mask(cfg).astype(np.uint8)).to(device)
        keep = {cfg.lp_etype: k}
        if cfg.lp_rev_etype >= 0:
            keep[cfg.lp_rev_etype] = k
    part_topo = partition is not None and topology == "partitioned"
    if part_topo:
        from paper_2406_06022_b200.dist import balanced_bounds
        pb = balanced_bounds(cfg.counts, partition[0])
    for r in range(cfg.num_etypes):
        if part_topo and keep is None:
            # synthetic input generation in edge chunks, keeping this rank's dst range only (a
            # rank never holds the whole COO: 2.16B edges for MAG240M, 10B for synth_10b); the
            # global CSC position of the range's first edge = the edges with a smaller dst
            t = int(cfg.etypes[r].dst)
            lo, hi = int(pb[t][partition[1]]), int(pb[t][partition[1] + 1])
            E = cfg.etypes[r if cfg.etypes[r].reverse_of is None else cfg.etypes[r].reverse_of].num_edges
            ss, dd, before = [], [], 0
            for a in range(0, E, 1 << 28):
                s, d = synth.etype_coo(cfg, r, backend="torch", device=device, lo=a, hi=min(E, a + (1 << 28)))
                m = (d >= lo) & (d < hi)
                before += int((d < lo).sum().item())
                ss.append(s[m])
                dd.append(d[m])
                del s, d, m
            s, d = torch.cat(ss), torch.cat(dd)
            del ss, dd
            st.load_etype_range(r, s, d, lo, hi, eid_base=before)
        elif part_topo:
            s, d = synth.etype_coo(cfg, r, backend="torch", device=device)
            t = int(cfg.etypes[r].dst)
            st.load_etype_range(r, s, d, int(pb[t][partition[1]]), int(pb[t][partition[1] + 1]),
                                None if keep is None else keep.get(r))
        else:
            s, d = synth.etype_coo(cfg, r, backend="torch", device=device)
            st.load_etype(r, s, d, None if keep is None else keep.get(r))
        del s, d
        torch.cuda.empty_cache()
    if part_topo:
        from paper_2406_06022_b200.dist import PeerCSC
        st._peer_csc = PeerCSC(st, partition[0], partition[1], pb, map_peers=(sampling == "peer"))
    ex = None
    if partition is None:
        for t in range(cfg.num_ntypes):
            st.set_features(t, synth.feature_table(cfg, t, backend="torch", device=device))
    else:
        from paper_2406_06022_b200.dist import FeatureExchange, PeerFeatures, balanced_bounds
        world, rank = partition
        b = balanced_bounds(cfg.counts, world)
        tdt = torch.bfloat16 if cfg.feat_dtype == "bf16" else torch.float32
        shards = [synth.feature_table(cfg, t, "torch", device, lo=int(b[t][rank]), hi=int(b[t][rank + 1]))
                  for t in range(cfg.num_ntypes)]
        if mode == "peer":
            st._peer = PeerFeatures(st, cfg.counts, world, rank, shards, cfg.feat_dim)
        else:
            ex = FeatureExchange(cfg.counts, world, rank, shards, cfg.feat_dim)
            st.feat_dim = cfg.feat_dim
            st.feat_dtype = tdt
    torch.cuda.synchronize()
    if cfg.task == "lp":
        local = None
        if LP_OPTS["neg"] == "local_joint" and partition is not None:
            from paper_2406_06022_b200.dist import balanced_bounds
            world, rank = partition
            dt = cfg.etypes[cfg.lp_etype].dst
            b = balanced_bounds(cfg.counts, world)
            local = (int(b[dt][rank]), int(b[dt][rank + 1] - b[dt][rank]))
        names = [k for k in synth.param_order(cfg) if LP_OPTS["score"] == "distmult" or k != "rel"]
        tr = LPTrainer(st, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_neg, cfg.lp_etype, cfg.lp_rev_etype,
                       {k: v for k, v in synth.init_params(cfg).items() if k in names}, names, lr=cfg.lr,
                       rng_seed=cfg.rng_seed, neg_sampler=LP_OPTS["neg"], score=LP_OPTS["score"], local_range=local)
    else:
        tr = RGCNTrainer(st, cfg.fanouts, cfg.batch, cfg.hidden, cfg.num_classes, synth.init_params(cfg),
                         synth.param_order(cfg), synth.labels(cfg, backend="torch", device=device),
                         int(cfg.node_off[cfg.target_ntype]), lr=cfg.lr, rng_seed=cfg.rng_seed)
    if LP_OPTS["learnable_emb"] and getattr(tr, "enc_types", None):
        for t in range(cfg.num_ntypes):
            if not cfg.project[t]:     # init = the frozen table, widened to fp32
                E = synth.feature_table(cfg, t, backend="torch", device=device).float()
                pe = None
                if partition is not None and partition[0] > 1:   # N > 1: partitioned over the ranks
                    from paper_2406_06022_b200.dist import PeerEmbedding
                    pe = PeerEmbedding(E, partition[0], partition[1])
                    tr._peer_emb = getattr(tr, "_peer_emb", []) + [pe]
                tr.set_embedding(t, E, peers=pe)
                del E
    tr.exchange = ex
    if part_topo and sampling == "nccl":
        from paper_2406_06022_b200.dist import SampleExchange
        tr._sx = SampleExchange(tr.sampler, partition[0], partition[1], first_hop=1)
    return st, tr


def poll_all(tr):
    """Poll the device error words of every sampler (both pipeline buffers).  Each word is
    sticky (OR of every sample since the last poll), so one poll after a timed loop covers
    all of its steps."""
    samplers = [tr.sampler]
    for b in (tr._bufs or []):
        if b["sampler"] not in samplers:
            samplers.append(b["sampler"])
    for sm in samplers:
        code = sm.poll_error()
        if code != 0:
            raise RuntimeError(f"device-side sampling error {code} latched")


_GRAPH_LAUNCHES = {}


def launches_per_step_graph(tr, cfg):
    """libgsb kernels in one captured step (counted once while capturing an eager twin)."""
    from paper_2406_06022_b200 import _lib
    key = id(tr)
    if key not in _GRAPH_LAUNCHES:
        _GRAPH_LAUNCHES[key] = tr.graph_launches
    return _GRAPH_LAUNCHES[key]


def block_sizes(tr, cfg):
    L = len(cfg.fanouts)
    sm = tr.sampler
    out = {"n_dst": [], "n_src": [], "n_edges": [], "acat_cols": [], "src_type_cnt0": None, "nonempty_segs": [],
           "dst_rel": [], "src_gid0": None}
    slots = tr.store.slot_etypes()
    for l in range(L):
        b = sm.block(l)
        d = cfg.feat_dim if l == 0 else cfg.hidden
        out["n_dst"].append(int(b.dst_gid.numel()))
        out["n_src"].append(int(b.src_gid.numel()))
        out["n_edges"].append(int(b.e_src.numel()))
        out["acat_cols"].append(int(sum(int(b.dst_type_cnt[t]) * (len(slots[t]) + 1) * d for t in range(len(slots)))))
        out["nonempty_segs"].append(int((b.seg_ptr[1:] > b.seg_ptr[:-1]).sum().item()))
        out["dst_rel"].append(int(sum(int(b.dst_type_cnt[t]) * len(slots[t]) for t in range(len(slots)))))
        if l == 0:
            out["src_gid0"] = b.src_gid.cpu().numpy()
        if l == 0:
            out["src_type_cnt0"] = [int(x) for x in b.src_type_cnt]
    return out


def run_gsb(args, cfg):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = f"cuda:{local}"
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(device))
    from paper_2406_06022_b200 import _lib
    t0 = time.time()
    if args.sampling == "nccl":
        args.features = "alltoall"
    partitioned = dist is not None and args.features != "replicate"
    st, tr = build_gsb(cfg, device, (ws, rank) if partitioned else None, args.features, args.topology,
                       args.sampling)
    if partitioned and args.features == "peer" and args.peer_gather == "unique":
        tr.fuse_gather = False   # unique rows over NVLink once (peer loads bypass L2), then local aggregation
    setup_s = time.time() - t0
    n_batches = args.warmup + args.steps + args.profile_steps + 8
    local_seeds = ws > 1 and partitioned and args.topology == "partitioned"
    if cfg.task == "lp":
        lpb = synth.LPBatcher(cfg)
        uv = [lpb.batch((i * ws + rank) % 100000) for i in range(n_batches)]
        us_all = torch.from_numpy(np.stack([x[0] for x in uv])).to(device)
        vs_all = torch.from_numpy(np.stack([x[1] for x in uv])).to(device)
        host_batches = [np.stack([x[0], x[1]]) for x in uv[:args.steps + 1]]
    else:
        train = synth.train_nodes(cfg)
        if local_seeds:
            # partitioned graph: every rank iterates over the training nodes it owns (DistDGL-style
            # locality, SURVEY §8(e) "NC: each GPU takes seeds from its own training nodes"), so
            # the seeds' own segments and rows are local; batch b of rank r = slice b of its epoch
            # permutation, RNG step word b * ws + r (globally unique)
            from paper_2406_06022_b200.dist import balanced_bounds
            bt = balanced_bounds(cfg.counts, ws)[cfg.target_ntype]
            loc = train - cfg.node_off[cfg.target_ntype]
            train = train[(loc >= bt[rank]) & (loc < bt[rank + 1])]
            per_epoch = max(1, len(train) // cfg.batch)
            bidx = lambda i: i % (per_epoch * 4)
        else:
            per_epoch = max(1, len(train) // cfg.batch)
            bidx = lambda i: (i * ws + rank) % (per_epoch * 4)
        # seed batches (a1): device-resident epoch permutation slices; rank r takes batch step*ws + r
        seeds_all = torch.from_numpy(np.stack([synth.nc_seeds(cfg, bidx(i), train)
                                               for i in range(n_batches)])).to(device)
        host_batches = [synth.nc_seeds(cfg, bidx(i), train) for i in range(args.steps + 1)]

    def fb(i):
        if cfg.task == "lp":
            tr.forward_backward(us_all[i], vs_all[i], i * ws + rank)
        else:
            tr.forward_backward(seeds_all[i], i * ws + rank)

    def load(i):
        if cfg.task == "lp":
            tr.load_inputs(us_all[i], vs_all[i])
        else:
            tr.load_inputs(seeds_all[i])

    def step(i):
        fb(i)
        if dist is not None:
            allreduce(tr.grad)                # C6: NCCL all-reduce (ncclAvg) of the flat dense grads
        tr.optimizer_step()

    def allreduce(g):
        from paper_2406_06022_b200.dist import allreduce_mean
        allreduce_mean(g)

    W = max(args.warmup, 3)
    for i in range(W - 2):
        step(i)
    torch.cuda.synchronize()
    poll_all(tr)
    # ---- CUDA graphs.  Pipelined (default): per-buffer graphs of the sample phase (side
    # stream, batch i+1) and of the compute phase (+ Adam) of batch i; otherwise ONE graph of
    # the whole step.  Replays advance the RNG step word and Adam's t on the device; inputs
    # are copied into the graphs' fixed buffers.
    # all-to-all exchange modes (host-synced sizes): only the pipelined path, whose sample phase
    # then runs eagerly beside the captured compute graph
    use_graph = not args.no_graph and (tr.exchange is None or args.pipeline == "on")
    pipelined = use_graph and args.pipeline == "on"

    def inputs(i):
        return (us_all[i], vs_all[i]) if cfg.task == "lp" else (seeds_all[i],)

    ar = allreduce if dist is not None else None
    if pipelined:
        tr.pipeline_start(inputs(W - 2), (W - 2) * ws + rank, ws=ws, allreduce=ar)
    elif use_graph:
        load(W - 2)
        tr.capture(step0=(W - 2) * ws + rank, ws=ws, allreduce=ar)

    def run(i):
        if pipelined:
            tr.pipeline_step(*inputs(i + 1))
        elif use_graph:
            load(i)
            tr.replay()
        else:
            step(i)

    for i in range(W - 2, W):
        run(i)
    torch.cuda.synchronize()
    poll_all(tr)
    # ---- timed region
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.lib().gsb_launch_count()
    if tr.exchange is not None:
        tr.exchange.bytes_sent = 0
    # frontier exchanges: one per pipeline buffer's sampler (MiniBatchSampler.twin attaches its own)
    sxs = [b["sampler"]._sx for b in (tr._bufs or []) if getattr(b["sampler"], "_sx", None) is not None] \
        or ([tr._sx] if getattr(tr, "_sx", None) is not None else [])
    for sx in sxs:
        sx.bytes_sent = 0
        sx.host_s = {}
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record()
        th0 = time.perf_counter()
        for i in range(W, W + args.steps):
            run(i)
        if pipelined:
            tr.pipeline_sync()    # the sampling of batch W+steps (issued in the last step) is inside
        e1.record()
        host_enqueue_ms = (time.perf_counter() - th0) * 1e3
        torch.cuda.synchronize()
    poll_all(tr)     # sticky latch: any sampling error in any timed step fails the run
    if dist is not None:
        dist.barrier()
    launches = _lib.lib().gsb_launch_count() - launches0
    nv_bytes = tr.exchange.bytes_sent / args.steps if tr.exchange is not None else 0
    nv_bytes += sum(sx.bytes_sent for sx in sxs) / args.steps      # C2/C3 frontier exchange
    if sxs and os.environ.get("GSB_XPROF") and rank == 0:
        tot = {}
        for sx in sxs:
            for k, v in sx.host_s.items():
                tot[k] = tot.get(k, 0.0) + v
        print("[xprof] host ms per step in the exchange callbacks (timed region):",
              {k: round(v * 1e3 / max(args.steps, 1), 3) for k, v in tot.items()}, "host enqueue ms/step",
              round(host_enqueue_ms / args.steps, 3), file=sys.stderr)
    if use_graph:   # kernels inside a replayed graph are not re-counted by the library
        eager = launches if (pipelined and tr.pipe_graphs and tr.pipe_graphs.get("sample") is None) else 0
        launches = launches_per_step_graph(tr, cfg) * args.steps + eager   # + eager sample-phase kernels
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    seeds_per_s = cfg.batch * ws * args.steps / (ms / 1e3)   # NC: seeds; LP: positive edges

    # ---- phase diagnostic: the pipelined step overlaps a sample-phase graph (side stream)
    # with a compute-phase graph; replayed alone, each one's time shows which bounds the step
    phase_ms = None
    if pipelined and getattr(tr, "pipe_graphs", None):
        torch.cuda.synchronize()
        phase_ms = {}
        for kind in ("sample", "compute"):
            if tr.pipe_graphs.get(kind) is None:   # eager sample phase (host-synced exchanges)
                continue
            g = tr.pipe_graphs[kind][0]
            tr._use(0)
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            phase_ms[kind] = a.elapsed_time(b) / 20
        if dist is not None:
            for k in list(phase_ms):
                t = torch.tensor([phase_ms[k]], device=device)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                phase_ms[k] = float(t.item())

    # ---- per-kernel profile: eager steps, each preceded by a 3 ms spin kernel so the host
    # enqueues the whole step before it starts (events then time kernels, not launch gaps)
    base = W + args.steps
    import ctypes as C
    _lib.lib().gsb_profile_enable(1)
    for i in range(base, base + args.profile_steps):
        _lib.call("gsb_spin", 3_000_000, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        step(i)
    torch.cuda.synchronize()
    _lib.lib().gsb_profile_enable(0)
    # block sizes of the profiled steps: sampling is a pure function of (seeds, step), so
    # re-sampling the same batches reproduces them bit-exactly
    sizes = []
    for i in range(base, base + args.profile_steps):
        if cfg.task == "lp":
            fb(i)          # sampling inputs depend on the negatives/seeds of the step
        else:
            tr.sampler.sample(seeds_all[i], tr.rng_seed, i * ws + rank)
        sizes.append(block_sizes(tr, cfg))
    buf = C.create_string_buffer(1 << 16)
    if os.environ.get("GSB_TIMELINE"):   # tools: per-launch timeline of the profiled steps
        tl = C.create_string_buffer(1 << 20)
        _lib.call("gsb_profile_timeline", tl, len(tl))
        with open(os.environ["GSB_TIMELINE"], "w") as f:
            f.write(tl.value.decode())
    _lib.call("gsb_profile_dump", buf, len(buf))
    prof = {}
    for line in buf.value.decode().splitlines():
        n, c, t = line.split()
        if n == "spin":
            continue
        prof[n] = {"launches": int(c), "total_ms": float(t)}
    edges_per_step = float(np.mean([sum(s["n_edges"]) for s in sizes]))
    # ---- e2e: public API with host buffers (pinned seeds H2D + loss D2H every step)
    host_pinned = [torch.from_numpy(b).pin_memory() for b in host_batches]
    # every step's loss is copied to pinned host memory and read by the host one step later
    # (event of step i-1 waited on after step i is enqueued): the usual asynchronous logging
    # loop, so the host never drains the device between steps
    loss_host = torch.zeros(args.steps, dtype=torch.float32).pin_memory()
    loss_ev = [torch.cuda.Event() for _ in range(args.steps)]
    losses_read = []
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if pipelined:   # prologue (first batch H2D + sampling) inside the timed region
        tr.pipeline_start(tuple(host_pinned[0]) if cfg.task == "lp" else (host_pinned[0],), base * ws + rank,
                          ws=ws, allreduce=ar)
    for i in range(args.steps):
        hb = host_pinned[i]
        if pipelined:
            nb = host_pinned[i + 1]
            tr.pipeline_step(*(tuple(nb) if cfg.task == "lp" else (nb,)))
        elif cfg.task == "lp":
            tr.pos_u.copy_(hb[0], non_blocking=True)
            tr.pos_v.copy_(hb[1], non_blocking=True)
        else:
            tr.seeds_dev[:hb.numel()].copy_(hb, non_blocking=True)
        if pipelined:
            pass
        elif use_graph:
            tr.replay()
        else:
            if cfg.task == "lp":
                tr._step_body(None, base + i)
            else:
                tr.forward_backward(tr.seeds_dev[:hb.numel()], base + i)
            if dist is not None:
                allreduce(tr.grad)
            tr.optimizer_step()
        loss_host[i:i + 1].copy_(tr.loss, non_blocking=True)
        loss_ev[i].record()
        if i >= 1:
            loss_ev[i - 1].synchronize()
            losses_read.append(float(loss_host[i - 1]))
    if pipelined:
        tr.pipeline_sync()
    torch.cuda.synchronize()
    losses_read.append(float(loss_host[args.steps - 1]))
    e2e_s = time.perf_counter() - t0
    poll_all(tr)
    if dist is not None:
        t = torch.tensor([e2e_s], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": cfg.batch * ws * args.steps / e2e_s, "unit": UNIT if cfg.task == "nc" else "pos_edges/s",
           "h2d_bytes_per_step": int(host_pinned[0].numel() * 8), "d2h_bytes_per_step": 4,
           "final_loss": losses_read[-1], "loss_reads": len(losses_read),
           "host_read": "every step's loss D2H into pinned memory, read on the host one step later"}
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None
    # ---- roofline of the dominant kernel (the most expensive one with an algorithmic-work
    # model) and, separately, of the fused gather + aggregation (north_star target)
    pk = peaks()
    ranked = [k for k, _ in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"])]
    dom = next((k for k in ranked if kernel_work(k, sizes[0], cfg)[0] is not None), ranked[0])
    roof = roofline_of(dom, prof, sizes, cfg, pk, args.profile_steps)
    roof_agg = roofline_of("rgcn_agg_l0", prof, sizes, cfg, pk, args.profile_steps) if "rgcn_agg_l0" in prof else None
    roof_more = {}
    for k in ranked:
        if k == dom or k == "rgcn_agg_l0":
            continue
        e = roofline_of(k, prof, sizes, cfg, pk, args.profile_steps)
        if e is not None:
            roof_more[k] = {x: e[x] for x in ("bound", "achieved", "peak", "unit", "frac", "avg_launch_us",
                                               "launches_per_step", "traffic", "dram_frac") if x in e}
    nvlink = None
    if ws > 1 and args.features == "peer":
        # unique input rows owned by other ranks, fetched over NVLink (peer loads) per step; the
        # remote CSC segments the sampler reads are small next to them (16 B indptr + f x 4 B)
        from paper_2406_06022_b200.dist import balanced_bounds
        bnd = balanced_bounds(cfg.counts, ws)
        rem = []
        for sz in sizes:
            g0 = sz["src_gid0"]
            t = np.searchsorted(cfg.node_off, g0, side="right") - 1
            loc = g0 - cfg.node_off[t]
            own = (loc >= bnd[t, rank]) & (loc < bnd[t, rank + 1])
            rem.append(int((~own).sum()))
        rbytes = float(np.mean(rem)) * cfg.feat_dim * (2 if cfg.feat_dtype == "bf16" else 4)
        k = "gather" if "gather" in prof else "rgcn_agg_l0"
        kus = prof[k]["total_ms"] / args.profile_steps * 1e3 if k in prof else None
        nvlink = {"kernel": k, "remote_rows_per_step": float(np.mean(rem)), "bytes_per_step": rbytes,
                  "achieved": rbytes / (kus / 1e6) / 1e9 if kus else None, "peak": 900.0, "unit": "GB/s",
                  "frac": (rbytes / (kus / 1e6) / 1e9 / 900.0) if kus else None,
                  "peak_src": "NVLink 5 per-direction bandwidth per GPU (B200_PROFILING.md)",
                  "note": "bytes the kernel pulls from peer HBM / its CUDA-event time in the profiled steps"}
    step_ms_prof = sum(v["total_ms"] for v in prof.values()) / args.profile_steps
    kernels = {k: {"us_per_step": v["total_ms"] * 1e3 / args.profile_steps,
                   "share": v["total_ms"] / args.profile_steps / step_ms_prof} for k, v in
               sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"])}
    topo = ("CSC partitioned by dst node ID, remote segments read over NVLink by the sampling kernels"
            if args.topology == "partitioned" and args.features != "replicate" else "topology replicated")
    if args.sampling == "nccl" and args.topology == "partitioned":
        topo = ("CSC partitioned by dst node ID, frontier sent to the owners and sampled edges returned by NCCL "
                "all-to-alls (C2/C3, owner-side keyed sampling)")
    par = ("single" if ws == 1 else {
        "peer": f"dp{ws}: features partitioned by node ID, read over NVLink (CUDA IPC) by libgsb kernels "
                f"({args.peer_gather} gather); {topo}; NCCL mean all-reduce of the grads after the CUDA graph",
        "alltoall": f"dp{ws}: features partitioned by node ID, NCCL all-to-all fetch; {topo}; "
                    f"NCCL mean all-reduce of the grads",
        "replicate": f"dp{ws}: graph + features replicated, NCCL grad all-reduce"}[args.features])
    unit = UNIT if cfg.task == "nc" else "pos_edges/s"
    metric = METRIC if cfg.task == "nc" else "RGCN LP train positive edges/sec on B200"
    line = {
        "metric": metric, "value": seeds_per_s, "unit": unit, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if cfg.feat_dtype == "f32" else "f32 (bf16 feature storage)", "data": "synthetic (seeded hash generator, synth/)",
        "config": cfg_json(cfg, ws, {"parallelism": par, "cuda_graph": use_graph,
                                     "seeds": ("each rank's batches are slices of its own training nodes (owner-local)"
                                               if cfg.task == "nc" and local_seeds else "global epoch permutation"),
                                     "pipeline": "sample i+1 on a side stream during compute i" if pipelined
                                     else "off"}),
        "sampled_edges_per_s": edges_per_step * ws / (ms_per_step / 1e3),
        "clocks": clk.summary(), "e2e": e2e, "gpu_launches": int(launches), "roofline": roof,
        "roofline_gather_aggregation": roof_agg,
        "roofline_kernels": roof_more,
        "nvlink": nvlink,
        "kernels": kernels, "setup_s": setup_s,
        "phase_ms_alone": phase_ms,
        "host_enqueue_ms_per_step": host_enqueue_ms / args.steps,
    }
    if tr.exchange is not None:
        line["nvlink_bytes_per_step_rank0"] = nv_bytes
    if dist is not None:
        dist.destroy_process_group()
    return line, st, tr


# ------------------------------------------------------------------------------ oracle
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_rate(cfg, seconds: float, sub_batch: int, max_steps: int = 10 ** 9, min_steps: int = 1):
    """Time the oracle (as it stands) on bounded samples of the workload: train steps on
    sub-batches of `sub_batch` seeds, first single-threaded, then on all host cores
    (oracle_set_threads: the layer loops over OpenMP threads, bit-identical results), each
    for about seconds/2 of CPU work.  value = the all-core rate."""
    import oracle
    t0 = time.time()
    og = oracle.Graph(cfg)
    if not cfg.has_encoder:   # encoder configs read rows from the generator's closed form
        for t in range(cfg.num_ntypes):
            og.feats[t] = synth.feature_table(cfg, t)
    setup = time.time() - t0
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    opt = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    labels = synth.labels(cfg)
    train = synth.train_nodes(cfg)
    nproc = os.cpu_count() or 1
    rates = {}
    step_i = 0
    for threads in (1, nproc):
        oracle.set_threads(threads)
        n_seeds, steps, el = 0, 0, 0.0
        while (el < seconds / 2 or steps < min_steps) and steps < max_steps:
            seeds = synth.nc_seeds(cfg, step_i, train)[:sub_batch]
            t1 = time.perf_counter()
            oracle.train_step(og, params, opt, step_i + 1, (seeds, labels), step_i, cfg.rng_seed, cfg.lr)
            el += time.perf_counter() - t1
            n_seeds += len(seeds)
            steps += 1
            step_i += 1
        rates[threads] = (n_seeds / el, steps, el)
    oracle.set_threads(1)
    v1, s1, e1 = rates[1]
    vn, sn, en = rates[nproc]
    return {"value": vn, "unit": UNIT, "cores": nproc, "kind": "oracle",
            "sample": f"oracle train steps of {sub_batch} seeds each ({cfg.name} graph, fanouts {cfg.fanouts}): "
                      f"{sn} steps in {en:.1f} s on {nproc} threads (OpenMP over dst rows, bit-identical), "
                      f"{s1} steps in {e1:.1f} s on 1 thread; oracle CSC build {setup:.1f} s excluded",
            "value_1thread": v1, "nproc": nproc, "cpu_model": cpu_model(), "steps": sn + s1,
            "seconds": en + e1}


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    sub = max(8, cfg.batch // 16)
    import oracle
    nproc = os.cpu_count() or 1
    oracle.set_threads(nproc)          # the oracle as it stands, on all host cores (bit-identical)
    t0 = time.time()
    og = oracle.Graph(cfg)
    if not cfg.has_encoder:   # encoder configs read rows from the generator's closed form
        for t in range(cfg.num_ntypes):
            og.feats[t] = synth.feature_table(cfg, t)
    setup = time.time() - t0
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    opt = {k: {"m": np.zeros_like(v), "v": np.zeros_like(v)} for k, v in params.items()}
    labels = synth.labels(cfg)
    train = synth.train_nodes(cfg)

    def step(i):
        seeds = synth.nc_seeds(cfg, i, train)[:sub]
        oracle.train_step(og, params, opt, i + 1, (seeds, labels), i, cfg.rng_seed, cfg.lr)

    for i in range(args.warmup):
        step(i)
    t1 = time.perf_counter()
    for i in range(args.warmup, args.warmup + args.steps):
        step(i)
    el = time.perf_counter() - t1
    v = sub * args.steps / el
    return {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded hash generator, synth/)", "impl": "reference",
            "config": cfg_json(cfg, ws, {"reference_sub_batch": sub}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nproc, "kind": "oracle",
                             "sample": f"each step = one oracle train step on {sub} of the batch's seeds, "
                                       f"{nproc} OpenMP threads; oracle CSC build {setup:.1f} s excluded",
                             "cpu_model": cpu_model(), "nproc": nproc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


def main():
    args = parse()
    cfg = config_for(args.config)
    LP_OPTS.update(neg=args.neg, score=args.score, learnable_emb=args.learnable_emb)
    fd = args.feat_dtype
    if fd == "auto":
        fd = cfg.feat_dtype if cfg.name in ("tiny", "tiny_lp") or cfg.feat_dtype == "bf16" else "bf16"
    cfg = synth.with_dtype(cfg, fd)
    if args.impl == "reference":
        line = run_reference(args, cfg)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    out = run_gsb(args, cfg)
    if out is None:
        return
    line, st, tr = out
    # the oracle baseline: rank 0 at N=1 only, and only where the oracle can hold the graph
    if not args.no_cpu_baseline and cfg.task == "nc" and dist_env()[0] == 1 and cfg.num_edges <= 200_000_000:
        del tr, st
        import torch
        torch.cuda.empty_cache()
        line["cpu_baseline"] = oracle_rate(cfg, args.cpu_seconds, cfg.batch)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
