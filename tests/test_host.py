"""CPU tests of host-side pieces: the shared input generator (numpy and torch produce the
same bits, value ranges, power-law shape), the LP batch source, and the bench.py reference
arm's JSON-line contract."""
import json
import os
import subprocess
import sys

import numpy as np
import torch

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_generator_numpy_torch_bit_identical():
    for cfg in (synth.tiny(), synth.scaled(synth.mag(), 0.001), synth.tiny_lp()):
        for r in range(cfg.num_etypes):
            s, d = synth.etype_coo(cfg, r, hi=min(5000, cfg.etypes[r].num_edges))
            st, dt = synth.etype_coo(cfg, r, backend="torch", hi=min(5000, cfg.etypes[r].num_edges))
            assert np.array_equal(s, st.numpy()) and np.array_equal(d, dt.numpy())
            assert s.min() >= 0 and s.max() < cfg.counts[cfg.etypes[r].src]
            assert d.min() >= 0 and d.max() < cfg.counts[cfg.etypes[r].dst]
        ids = np.arange(0, cfg.counts[0], max(1, cfg.counts[0] // 97))
        f = synth.feature_rows(cfg, 0, ids)
        ft = synth.feature_rows(cfg, 0, torch.from_numpy(ids), backend="torch")
        assert np.array_equal(f, ft.numpy()) and f.min() >= -1.0 and f.max() < 1.0
        assert np.array_equal(synth.labels(cfg), synth.labels(cfg, backend="torch").numpy())


def test_bf16_features_are_rne_rounded_fp32_features():
    """bf16 feature storage: every value is the fp32 feature rounded to the
    nearest bf16 (ties to even) -- checked against torch's own conversion -- numpy and torch
    agree bit for bit, and the torch table converts to bfloat16 exactly."""
    cfg = synth.with_dtype(synth.tiny(), "bf16")
    ids = np.arange(0, 4000, 3)
    f32 = synth.feature_rows(synth.tiny(), 2, ids)
    bf = synth.feature_rows(cfg, 2, ids)
    assert np.array_equal(bf, torch.from_numpy(f32).to(torch.bfloat16).float().numpy())
    assert np.array_equal(bf, synth.feature_rows(cfg, 2, torch.from_numpy(ids), backend="torch").numpy())
    assert np.abs(bf - f32).max() <= 2.0 ** -8          # half an ulp of bf16 on [-1, 1)
    tab = synth.feature_table(cfg, 2, backend="torch")
    assert tab.dtype == torch.bfloat16
    assert np.array_equal(tab.float().numpy(), synth.feature_table(cfg, 2))
    # ties round to even: 1 + 2^-8 is halfway between bf16 neighbours 1 and 1 + 2^-7
    x = np.array([1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8], np.float32).view(np.uint32).astype(np.uint64)
    r = (synth._round_bf16_bits(x) & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)
    assert r[0] == 1.0 and r[1] == 1.0 + 2.0 ** -6


def test_reverse_etypes_mirror_forward():
    cfg = synth.mag()
    s, d = synth.etype_coo(cfg, 0, hi=1000)
    rs, rd = synth.etype_coo(cfg, 4, hi=1000)   # rev_writes
    assert np.array_equal(s, rd) and np.array_equal(d, rs)


def test_power_law_in_degree():
    """Degree profile of the Chung-Lu-style generator: heavy tail (max >> mean) and the rank
    mapping is a bijection (every id reachable)."""
    cfg = synth.tiny()
    s, d = synth.etype_coo(cfg, 0)
    deg = np.bincount(d, minlength=cfg.counts[0])
    assert deg.max() > 50 * deg.mean()
    a, b = synth._affine(cfg.counts[0], 0)
    ranks = np.arange(cfg.counts[0])
    assert len(np.unique((ranks * a + b) % cfg.counts[0])) == cfg.counts[0]


def test_lp_batcher_matches_reference_batches():
    cfg = synth.tiny_lp()
    b = synth.LPBatcher(cfg)
    keep = synth.lp_keep_mask(cfg)
    s, d = synth.etype_coo(cfg, cfg.lp_etype)
    train = set(zip((s[keep] + cfg.node_off[0]).tolist(), (d[keep] + cfg.node_off[0]).tolist()))
    for step in (0, 5):
        u, v = b.batch(step)
        u2, v2 = synth.lp_train_edges(cfg, step)
        assert np.array_equal(u, u2) and np.array_equal(v, v2)
        assert all((a_, b_) in train for a_, b_ in zip(u.tolist(), v.tolist()))


def test_nc_seeds_are_distinct_training_nodes():
    cfg = synth.tiny()
    tr = set(synth.train_nodes(cfg).tolist())
    for step in range(3):
        s = synth.nc_seeds(cfg, step)
        assert len(s) == cfg.batch and len(set(s.tolist())) == cfg.batch
        assert all(int(x) in tr for x in s)


def test_bench_reference_arm_json_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "tiny",
                          "--steps", "3", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e", "gpu_launches"):
        assert k in j, k
    assert j["impl"] == "reference" and j["steps"] == 3 and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["kind"] == "oracle"
