"""Host logic of bench.py (no GPU): the roofline object for every path and the
reference arm's JSON line (the CPU oracle on a bounded sample)."""
import importlib.util
import json
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def cfg_of(name):
    sys.path.insert(0, ROOT)
    from synth import configs
    return configs.ALL[name]


PEAK = 6552.6


def check(r, alg, ms, cfg, ms_step, n_hash):
    """Dominant kernel: SURVEY §8(d) algorithmic bytes per launch over its mean
    launch time; the step: |A| + |b| + |SA| + |Sb| + s 5 B per hashed row over
    the step time, against the measured peak and the 8 TB/s spec."""
    assert r["unit"] == "GB/s" and r["bound"] == "hbm" and r["peak"] == PEAK
    assert r["alg_bytes_per_launch"] == alg
    assert abs(r["achieved"] - alg / (ms / 1e3) / 1e9) <= 0.1
    assert abs(r["frac"] - r["achieved"] / PEAK) <= 1e-3
    assert abs(r["frac_of_8tbs_spec"] - r["achieved"] / 8000.0) <= 1e-3
    alg_step = cfg.a_bytes + cfg.n * 8 + cfg.m * cfg.d * 8 + cfg.m * 8 + n_hash * cfg.s * 5
    st = r["step"]
    assert st["alg_bytes"] == alg_step
    assert abs(st["alg_frac"] - alg_step / (ms_step / 1e3) / 1e9 / PEAK) <= 1e-4


def test_roofline_fwht_pass_counts_one_read_per_pass():
    """Judge's recomputation: an FWHT pass counts d 8 B per row,
    not the practical read + write; C5 0.49 at 21.354 ms, the step 0.142 at 74 ms."""
    b, cfg = bench(), cfg_of("C5")
    step = types.SimpleNamespace(plan=[7, 7, 7], n_pad=cfg.n)
    st = {"fork": 0.01, "fwht_pass0": 21.354, "fwht_pass1": 21.0, "fwht_pass2": 21.0, "gather": 9.7,
          "hash_gen (overlapped)": 0.13}
    r = b.roofline(cfg, step, st, 74.04, PEAK, "test")
    check(r, cfg.n * cfg.d * 8, 21.354, cfg, 74.04, cfg.n)
    assert r["stage"] == "fwht_pass0" and abs(r["frac"] - 0.4911) < 2e-3
    assert abs(r["step"]["alg_frac"] - 0.142) < 2e-3


def test_roofline_gather_csr_and_dht():
    b = bench()
    c3 = cfg_of("C3")
    r = b.roofline(c3, None, {"hash_gen": 0.06, "gather": 0.95}, 1.01, PEAK, "test")
    check(r, c3.n * c3.d * 8 + c3.m * c3.d * 8 + c3.n * c3.s * 5, 0.95, c3, 1.01, c3.n)
    assert r["kernel"] == "gather_group_kernel<16>"  # s = 2: the L2-slice kernel
    c4 = cfg_of("C4")
    r = b.roofline(c4, None, {"hash_gen": 0.14, "gather_csr": 0.57}, 0.72, PEAK, "test")
    check(r, c4.n * c4.nnz_row * 12 + (c4.n + 1) * 8 + c4.m * c4.d * 8 + c4.n * c4.s * 5, 0.57, c4, 0.72, c4.n)
    c2 = cfg_of("C2")
    st = {"hash_gen": 0.03, "dht_passA": 0.25, "dht_passB": 0.20, "gather": 0.11}
    r = b.roofline(c2, types.SimpleNamespace(n_pad=c2.n), st, 0.6, PEAK, "test", sketch="dht")
    check(r, c2.n * (c2.d + 1) * 8, 0.25, c2, 0.6, c2.n)
    assert r["stage"] == "dht_passA"


def test_roofline_column_major_paths():
    b = bench()
    c5 = cfg_of("C5")
    step = types.SimpleNamespace(n_pad=c5.n)
    st = {"hash_gen": 0.1, "tile_lists": 0.04, "pass1": 24.0, "pass2_gather": 23.0}
    r = b.roofline(c5, step, st, 47.3, PEAK, "test", layout="col")
    check(r, c5.n * (c5.d + 1) * 8, 24.0, c5, 47.3, c5.n)
    assert r["stage"] == "pass1"
    st["pass2_gather"] = 25.0
    r = b.roofline(c5, step, st, 49.3, PEAK, "test", layout="col")
    cols = c5.d + 1
    check(r, c5.n * cols * 8 + c5.m * cols * 8 + c5.n * c5.s * 5, 25.0, c5, 49.3, c5.n)
    c3 = cfg_of("C3")
    st = {"hash_gen": 0.06, "transpose": 1.55, "gather": 1.05}
    r = b.roofline(c3, types.SimpleNamespace(n_pad=c3.n), st, 2.7, PEAK, "test", layout="col")
    check(r, c3.n * c3.d * 8, 1.55, c3, 2.7, c3.n)
    assert "transpose" in r["kernel"]


def test_default_layout():
    """Column-major (the paper's layout) for H D workloads where the row-major
    plan needs >= 3 transform passes (C5, 21 stages) or s = 1 (C2); row-major
    otherwise."""
    b = bench()
    for name in ("C5", "C2"):
        assert b.default_layout(cfg_of(name)) == "col", name
    for name in ("C1", "C3", "C3HD", "C4"):
        assert b.default_layout(cfg_of(name)) == "row", name


@pytest.mark.timeout(600)
def test_reference_arm_json_line():
    """`bench.py --impl reference` (the CPU oracle) prints one JSON line with the
    contract's keys, on the C1 workload, without a GPU."""
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--workload", "C1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["config"]["workload"] == "C1"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
