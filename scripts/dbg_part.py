import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, oracle
from tests.test_gpu_partition_sim import partitioned_store
from paper_2406_06022_b200.dist import balanced_bounds
from paper_2406_06022_b200.runtime import MiniBatchSampler
world = int(sys.argv[1])
cfg = synth.with_dtype(synth.scaled(synth.mag(), 0.01, "mag_small"), "bf16")
st = partitioned_store(cfg, world)
og = oracle.Graph(cfg)
b = balanced_bounds(cfg.counts, world)
# shard CSC vs oracle slices (shards kept in st._keep: [indptr, indices] per (r, w) in order)
keep = st._keep[0]
k = 0
for r in range(cfg.num_etypes):
    t = cfg.etypes[r].dst
    for w in range(world):
        ip, ix = keep[k].cpu().numpy(), keep[k + 1].cpu().numpy(); k += 2
        lo, hi = b[t][w], b[t][w + 1]
        oip = og.indptr[r][lo:hi + 1] - og.indptr[r][lo]
        oix = og.indices[r][og.indptr[r][lo]:og.indptr[r][hi]]
        ok_ip = np.array_equal(ip, oip); ok_ix = np.array_equal(ix[:len(oix)], oix)
        if not (ok_ip and ok_ix):
            print("shard mismatch r", r, "w", w, ok_ip, ok_ix, len(ip), len(oip), len(ix), len(oix))
print("shards checked")
sm = MiniBatchSampler(st, [-1], max_seeds=cfg.num_nodes)
for t in range(cfg.num_ntypes):
    seeds = np.arange(cfg.node_off[t], cfg.node_off[t + 1], dtype=np.int64)[:int(sys.argv[2])]
    sm.sample(torch.from_numpy(seeds).cuda(), cfg.rng_seed, 0)
    torch.cuda.synchronize()
    gb = sm.block(0)
    ob = oracle.sample_blocks(og, seeds, [-1], cfg.rng_seed, 0)[0]
    g = gb.e_src_gid.cpu().numpy()
    bad = np.nonzero(g != ob.e_src_gid)[0]
    print("type", t, "edges", len(g), len(ob.e_src_gid), "bad", len(bad), "first", bad[:5], g[bad[:5]], ob.e_src_gid[bad[:5]])
    if len(bad):
        e = gb.e_eid.cpu().numpy()
        sp = gb.seg_ptr.cpu().numpy()
        i = np.searchsorted(sp, bad[0], side="right") - 1
        print("  seg", i, "range", sp[i], sp[i + 1], "eid got", e[bad[:5]], "exp", ob.e_eid[bad[:5]], "n_bad_in_seg",
              ((bad >= sp[i]) & (bad < sp[i + 1])).sum(), "first bad off in seg", bad[0] - sp[i])
