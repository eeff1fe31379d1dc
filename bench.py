#!/usr/bin/env python
"""Benchmark of the hashing-sketch hot path (BASELINE.json metric:
"sketch GB/s of A streamed (S.A, S.H.D.A) & % HBM peak at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5] [--layout row|col]
                    [--impl reference]

A step is one pass of the whole hot path over the workload (SURVEY §8(a) rows
R1-R5; R6/R7 as well when N > 1): hash_gen (draw S_h, bucket lists), the D +
Walsh-Hadamard passes, the bucket gather producing SA and Sb.  Default workload
C5 (BASELINE.json configs[4]: the config the metric is quoted on at 1/2/4/8
GPUs; it fits one B200).  Inputs are synthetic (synth/), generated on the
device and resident in HBM before timing; A (64 GiB) is larger than L2, so no
flush is needed.  Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the CPU oracle is timed single-threaded ("cores": 1 in cpu_baseline)
for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json: torch copy, read+write bytes)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------- CPU oracle (cpu_baseline / reference arm)
def oracle_sample(cfg, ncols):
    """Time the oracle as it stands on a bounded sample of the workload: ncols
    columns of A (all n rows), or a row block for CSR.  Returns (bytes, seconds, what)."""
    import numpy as np

    from oracle import sketch
    from synth import gen
    if cfg.kind == "csr":
        rows = max(1, int(cfg.n * ncols / 256))
        sub = cfg.scaled(n=rows)
        rp, ci, v = gen.csr(sub)
        b = gen.rhs(sub)
        t0 = time.perf_counter()
        sketch.sketch_csr(cfg.seed, rp, ci, v, cfg.d, b, cfg.m, cfg.s)
        t = time.perf_counter() - t0
        return rows * cfg.nnz_row * 12 + (rows + 1) * 8, t, f"CSR rows 0..{rows} of {cfg.name} (all buckets)"
    cols = list(range(ncols))
    Ablk = gen.dense_block(cfg, 0, cfg.n, cols)
    t0 = time.perf_counter()
    if cfg.hd:
        sketch.rht_sketch(cfg.seed, Ablk, None, cfg.m, cfg.s)
    else:
        sketch.sketch_dense(cfg.seed, Ablk, None, cfg.m, cfg.s)
    t = time.perf_counter() - t0
    del np
    return cfg.n * ncols * 8, t, f"{ncols} of {cfg.d} columns of {cfg.name} A, all {cfg.n} rows"


def cpu_baseline(cfg, target_s=12.0):
    """The oracle on a bounded column sample sized to ~target_s seconds: the
    per-sample fixed cost (drawing S for all n rows) is separated from the
    per-column cost with two probes, then the column count is chosen."""
    ncols = 1
    nbytes, t, what = oracle_sample(cfg, ncols)
    if t < target_s / 2 and cfg.kind != "csr":
        n2 = max(2, min(cfg.d, 4))
        nb2, t2, what2 = oracle_sample(cfg, n2)
        per_col = max((t2 - t) / (n2 - 1), 1e-4)
        fixed = max(t - per_col, 0.0)
        # host memory per sample: <= 512 MB of A under H D (its transform's temporaries), 1 GB plain
        cap = max(n2, ((512 << 20) if cfg.hd else (1 << 30)) // (cfg.n * 8))
        ncols = max(n2, min(cfg.d, cap, int((target_s - fixed) / per_col)))
        if ncols > n2 and t2 < target_s / 2:
            nbytes, t, what = oracle_sample(cfg, ncols)
        else:
            nbytes, t, what = nb2, t2, what2
    return {"value": nbytes / t / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{what}; {t:.2f} s single-threaded NumPy", "seconds": round(t, 3)}


def reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ncols = 2 if cfg.kind != "csr" else 4
    for _ in range(args.warmup):
        oracle_sample(cfg, ncols)
    tot_b, tot_t = 0, 0.0
    what = ""
    for _ in range(args.steps):
        nb, t, what = oracle_sample(cfg, ncols)
        tot_b += nb
        tot_t += t
    v = tot_b / tot_t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "d": cfg.d, "m": cfg.m, "s": cfg.s, "hd": cfg.hd,
                       "note": "CPU oracle on a bounded sample of the workload per step"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"{what} per step"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "sketch GB/s of A streamed (S.A, S.H.D.A) & % HBM peak"


# ---------------------------------------------------------------- GPU arm, one GPU
def build_step(cfg, torch, layout="row", sketch="hashing"):
    from paper_2105_11815_b200 import pipeline
    from synth import device
    var = sketch == "variant"
    if sketch in ("dht", "srdht"):
        A = device.dense(cfg)
        b = device.rhs(cfg)
        return pipeline.DhtStep(cfg.seed, A, b, cfg.m, cfg.s, sampling=sketch == "srdht", record=True), (A, b)
    if layout == "col" and cfg.kind != "csr":
        At = device.dense_colmajor(cfg)
        b = device.rhs(cfg)
        return pipeline.ColStep(cfg.seed, At, b, cfg.m, cfg.s, cfg.hd, record=True), (At, b)
    if cfg.kind == "csr":
        rp, ci, v = device.csr(cfg)
        b = device.rhs(cfg)
        return pipeline.CsrStep(cfg.seed, rp, ci, v, cfg.d, b, cfg.m, cfg.s, record=True, variant=var), (rp, ci, v, b)
    A = device.dense(cfg)
    b = device.rhs(cfg)
    cls = pipeline.HrhtStep if cfg.hd else pipeline.PlainStep
    return cls(cfg.seed, A, b, cfg.m, cfg.s, record=True, variant=var), (A, b)


def e2e_measure(cfg, inputs, steps, torch, layout="row"):
    """Same metric through the host-buffer C-ABI call: H2D of A and b and D2H of
    SA and Sb inside the timed region (pinned host buffers)."""
    import paper_2105_11815_b200 as skh
    if cfg.kind == "csr" or (layout == "col" and not cfg.hd):
        return None
    A, b = inputs
    A_h = torch.empty(A.shape, dtype=torch.float64, pin_memory=True)
    A_h.copy_(A)
    b_h = torch.empty(b.shape, dtype=torch.float64, pin_memory=True)
    b_h.copy_(b)
    torch.cuda.synchronize()
    if layout == "col":
        op = skh.RhtDenseColMajor(cfg.n, cfg.m, cfg.s, cfg.d)
        call = op.from_host
    elif cfg.hd:
        op = skh.RhtDense(cfg.n, cfg.m, cfg.s, cfg.d)
        call = op.from_host
    else:
        op = skh.SketchDenseHost(cfg.n, cfg.m, cfg.s, cfg.d)
        call = op
    SA_h = torch.empty(cfg.m, cfg.d, dtype=torch.float64, pin_memory=True)
    if layout == "col":
        SA_h = torch.empty(cfg.d, cfg.m, dtype=torch.float64, pin_memory=True)
    Sb_h = torch.empty(cfg.m, dtype=torch.float64, pin_memory=True)
    call(cfg.seed, A_h, b_h, SA_h, Sb_h)  # warm-up
    t = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        call(cfg.seed, A_h, b_h, SA_h, Sb_h)
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    del op
    ms = sum(t) / len(t)
    return {"value": cfg.a_bytes / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms, "steps": steps,
            "h2d_bytes_per_step": A.numel() * 8 + b.numel() * 8, "d2h_bytes_per_step": cfg.m * cfg.d * 8 + cfg.m * 8,
            "api": ("skh_rht_dense_colmajor_host" if layout == "col" else
                    "skh_rht_dense_host" if cfg.hd else "skh_sketch_dense_host")}


def roofline(cfg, step, stage_ms, peak_gbs, peak_src, layout="row", sketch="hashing"):
    """Dominant kernel and its algorithmic bytes per launch."""
    if sketch in ("dht", "srdht"):
        # stages of skh_hrdht_dense / skh_srdht_dense (row-major).  n = 2^L
        # (csrc/fht.cu): pass A reads D [A | b] and writes the half spectrum
        # (n/2 + n1 complex per column ~ the same bytes), pass B reads it and
        # writes the row-major transform.  Other n (or SKH_DHT_CUFFT=1): D +
        # transpose, cuFFT D2Z (a library FFT), Hartley combine + transpose.
        # Then the gather (or row sampling) reads the transform once.
        nb = cfg.n * (cfg.d + 1) * 8
        alg = {"diag": 2 * nb, "fft": 2 * nb, "hartley": 2 * nb, "dht_passA": 2 * nb, "dht_passB": 2 * nb,
               "gather": nb + cfg.m * cfg.d * 8 + cfg.n * cfg.s * 5}
        name = max((k for k in stage_ms if k in alg), key=lambda k: stage_ms[k])
        t = stage_ms[name]
        ach = alg[name] / (t / 1e3) / 1e9
        return {"bound": "hbm", "kernel": ("cufft D2Z (library)" if name == "fft" else name), "achieved": round(ach, 1),
                "peak": peak_gbs, "unit": "GB/s", "frac": round(ach / peak_gbs, 4), "traffic": None,
                "traffic_source": None, "alg_bytes_per_launch": alg[name], "ms_per_launch": round(t, 4),
                "peak_source": peak_src}
    if layout == "col" and "transpose" in stage_ms:
        # plain column-major sketch with the transposed path (skh.h): the tiled
        # transpose reads + writes A once; the row gather reads the copy once,
        # writes SA, and SA is transposed out (read + write)
        nb = cfg.n * cfg.d * 8
        alg = {"transpose": 2 * nb, "gather": nb + 3 * cfg.m * cfg.d * 8 + cfg.n * cfg.s * 5}
        label = {"transpose": "cm_to_rm_kernel (A transpose)", "gather": "gather_wide + SA transpose"}
        name = max((k for k in stage_ms if k in alg), key=lambda k: stage_ms[k])
        t = stage_ms[name]
        achieved = alg[name] / (t / 1e3) / 1e9
        return {"bound": "hbm", "kernel": label[name], "achieved": round(achieved, 1), "peak": peak_gbs,
                "unit": "GB/s", "frac": round(achieved / peak_gbs, 4), "traffic": None, "traffic_source": None,
                "alg_bytes_per_launch": alg[name], "ms_per_launch": round(t, 4), "peak_source": peak_src}
    if layout == "col":
        # dominant by time; algorithmic bytes of each kernel per launch:
        #  pass1: read + write (d + 1) columns of n_pad rows once
        #  pass2_gather / gather: read the columns once, write SA, read the tile lists
        cols = cfg.d + 1
        nrows = step.n_pad if cfg.hd else cfg.n
        lists = nrows * cfg.s * 4
        alg = {"pass1": 2 * step.n_pad * cols * 8,
               "pass2_gather": nrows * cols * 8 + cfg.m * cols * 8 + lists,
               "gather": nrows * cols * 8 + cfg.m * cols * 8 + lists}
        name = max((k for k in stage_ms if k in alg), key=lambda k: stage_ms[k])
        t = stage_ms[name]
        achieved = alg[name] / (t / 1e3) / 1e9
        traffic, tsrc = None, None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                ent = json.load(f).get(cfg.name + "-col")
            if ent and ent["kernel"] == "cm_" + name:
                traffic, tsrc = ent["dram_bytes_per_launch"], ent["source"]
        return {"bound": "hbm", "kernel": "cm_" + name, "achieved": round(achieved, 1), "peak": peak_gbs,
                "unit": "GB/s", "frac": round(achieved / peak_gbs, 4), "traffic": traffic, "traffic_source": tsrc,
                "alg_bytes_per_launch": alg[name], "ms_per_launch": round(t, 4), "peak_source": peak_src,
                "note": "bound on chip: the rank-round scatter into shared memory (DESIGN.md §5b); DRAM traffic "
                        "equals the algorithmic bytes"}
    if cfg.kind == "csr":
        name = "gather_csr"
        nnz = cfg.n * cfg.nnz_row
        alg = nnz * 12 + (cfg.n + 1) * 8 + cfg.m * cfg.d * 8 + cfg.n * cfg.s * 5
        t = stage_ms[name]
    elif cfg.hd:
        passes = [k for k in stage_ms if k.startswith("fwht_pass")]
        name = "fwht_tile_kernel (" + "+".join(str(k) for k in step.plan) + " stage passes, mean per launch)"
        alg = 2 * step.n_pad * cfg.d * 8          # read + write the n x d block once per pass
        t = sum(stage_ms[k] for k in passes) / len(passes)
    else:
        name = "gather_wide" if (cfg.d % 2 == 0 and cfg.d > 64) else "gather_dense"  # csrc/gather.cu kernel
        alg = cfg.n * cfg.d * 8 + cfg.m * cfg.d * 8 + cfg.n * cfg.s * 5
        t = stage_ms["gather"]
    achieved = alg / (t / 1e3) / 1e9
    traffic, tsrc = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            ent = json.load(f).get(cfg.name)
        if ent and ent["kernel"].split("<")[0] in name:
            traffic, tsrc = ent["dram_bytes_per_launch"], ent["source"]
    out = {"bound": "hbm", "kernel": name, "achieved": round(achieved, 1), "peak": peak_gbs, "unit": "GB/s",
           "frac": round(achieved / peak_gbs, 4), "traffic": traffic, "traffic_source": tsrc,
           "alg_bytes_per_launch": alg, "ms_per_launch": round(t, 4), "peak_source": peak_src}
    if achieved > peak_gbs:
        out["note"] = ("frac > 1: the peak is torch's device copy (b.copy_ of 2 GiB, best of 10); this pass "
                       "moves the same read + write bytes slightly faster")
    return out


def gpu_arm_single(args, cfg):
    import torch

    import paper_2105_11815_b200 as skh
    # the oracle sample runs first, while the host holds no pinned e2e buffers
    cpu_line = (cpu_baseline(cfg) if not args.no_cpu_baseline and args.sketch == "hashing" else None)
    torch.cuda.set_device(0)
    step, inputs = build_step(cfg, torch, args.layout, args.sketch)
    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 0)):
        step.run()
    torch.cuda.synchronize()
    timers = [step.new_timer() for _ in range(args.steps)]
    clk = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
    clk.start()
    time.sleep(0.3)
    n0 = skh.api.launch_count()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.steps):
        step.run(timers[k])
    e1.record()
    torch.cuda.synchronize()
    launches = skh.api.launch_count() - n0
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / args.steps
    per = [t.durations_ms() for t in timers]
    stage_ms = {k: sum(p[k] for p in per) / len(per) for k in per[0]}
    pk, src = peaks()
    value = cfg.a_bytes / (ms / 1e3) / 1e9
    line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "pct_hbm_peak": round(100 * value / pk["hbm_gbs"], 2),
            "config": {"workload": cfg.name, "n": cfg.n, "d": cfg.d, "m": cfg.m, "s": cfg.s, "hd": cfg.hd,
                       "a_bytes": cfg.a_bytes, "layout": "column-major" if args.layout == "col" else "row-major",
                       "l2": "inputs (A) larger than L2; no flush",
                       "parallelism": "single GPU", "note": cfg.note},
            "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
            "gpu_launches": int(launches), "clocks": clocks}
    line["roofline"] = roofline(cfg, step, stage_ms, pk["hbm_gbs"], src, args.layout, args.sketch)
    if args.sketch != "hashing":
        line["config"]["sketch"] = {"variant": "s-hashing variant (Def. 7)", "dht": "HR-DHT S_h F D (eq. (6.1))",
                                    "srdht": "SR-DHT S_s F D (eq. (7.2))"}[args.sketch]
    del step
    if not args.no_e2e:
        line["e2e"] = e2e_measure(cfg, inputs, args.e2e_steps, torch, args.layout) if args.sketch == "hashing" else None
    del inputs
    torch.cuda.empty_cache()
    if args.layout == "row" and cfg.kind != "csr" and cfg.hd and args.sketch == "hashing" and not args.no_alt_layout:
        line["column_major"] = alt_layout_measure(args, cfg, torch, pk, src)
        torch.cuda.empty_cache()
    if cpu_line is not None:
        line["cpu_baseline"] = cpu_line
    print(json.dumps(line), flush=True)


def alt_layout_measure(args, cfg, torch, pk, src):
    """The same workload stored column-major (the paper's LAPACK layout): the
    two-pass fused path of skh_rht_dense_colmajor, timed the
    same way; reported beside the row-major headline."""
    step, inputs = build_step(cfg, torch, "col")
    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 0)):
        step.run()
    timers = [step.new_timer() for _ in range(args.steps)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.steps):
        step.run(timers[k])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    per = [t.durations_ms() for t in timers]
    stage_ms = {k: sum(p[k] for p in per) / len(per) for k in per[0]}
    out = {"value": round(cfg.a_bytes / (ms / 1e3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
           "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
           "roofline": roofline(cfg, step, stage_ms, pk["hbm_gbs"], src, "col"),
           "note": "same A stored column-major; pass 1 (13 contiguous bits, D fused) + pass 2 fused with the "
                   "gather: 3|A| of HBM traffic vs 7|A|; SA to 1e-12 (DESIGN.md R17)"}
    del step, inputs
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--layout", default="row", choices=["row", "col"],
                    help="storage of dense A: row-major (default) or column-major (the paper's LAPACK layout)")
    ap.add_argument("--impl", default="skh", choices=["skh", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--sketch", default="hashing", choices=["hashing", "variant", "dht", "srdht"],
                    help="hashing (default, Def. 4 / HRHT), the s-hashing variant (Def. 7), HR-DHT (eq. 6.1) "
                         "or SR-DHT (eq. 7.2)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt-layout", action="store_true",
                    help="skip the column-major measurement reported beside a row-major H D workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    from synth import configs
    cfg = configs.ALL[args.workload]
    if args.impl == "reference":
        return reference_arm(args, cfg)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        if args.layout == "col":
            raise SystemExit("--layout col is single-GPU in this build (sharded runs use row-major A)")
        from paper_2105_11815_b200 import sharded_bench
        return sharded_bench.run(args, cfg)
    from paper_2105_11815_b200 import build
    build.build()
    return gpu_arm_single(args, cfg)


if __name__ == "__main__":
    main()
