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


SPEC_HBM_GBS = 8000.0  # B200 HBM3e spec sheet: the secondary denominator


def alg_bytes_step(cfg, n_hash):
    """SURVEY §8(d) algorithmic bytes of one whole step: read A (dense n d 8, or
    the CSR arrays) and b once, write SA and Sb once, plus s 5 bytes of bucket
    metadata (int32 row + int8 sign) per hashed row.  H D adds adds, not bytes."""
    return cfg.a_bytes + cfg.n * 8 + cfg.m * cfg.d * 8 + cfg.m * 8 + n_hash * cfg.s * 5


def kernel_table(cfg, step, layout, sketch):
    """Stage name -> (kernel, algorithmic bytes per launch, launches per step):
    per §8(d), a launch that reads X rows of A costs X d 8 bytes (a transform
    pass included: a fused transform would add none), a gather also writes SA
    and reads its bucket metadata."""
    if sketch in ("dht", "srdht"):
        nb = cfg.n * (cfg.d + 1) * 8
        return {"dht_passA": ("dht_passA_kernel", nb, 1), "dht_passB": ("dht_passB_kernel", nb, 1),
                "diag": ("diag_transpose", nb, 1), "fft": ("cufft D2Z (library)", nb, 1),
                "hartley": ("hartley combine", nb, 1),
                "gather": ("gather", nb + cfg.m * cfg.d * 8 + cfg.n * cfg.s * 5, 1)}
    if layout == "col" and cfg.kind != "csr":
        cols = cfg.d + 1
        if not cfg.hd:
            nb = cfg.n * cfg.d * 8
            return {"transpose": ("cm_to_rm_kernel (A transpose)", nb, 1),
                    "gather": ("gather_wide + SA transpose", nb + cfg.m * cfg.d * 8 + cfg.n * cfg.s * 5, 1)}
        npad = step.n_pad
        return {"pass1": ("cm_pass1_kernel", npad * cols * 8, 1),
                "mid_pass": ("cm_mid_kernel", npad * cols * 8, 1),
                "pass2_gather": ("cm_gather_kernel (fused last pass + owner-planned gather)",
                                 npad * cols * 8 + cfg.m * cols * 8 + npad * cfg.s * 5, 1)}
    if cfg.kind == "csr":
        return {"gather_csr": ("csr_expand + csr_reduce", cfg.a_bytes + cfg.m * cfg.d * 8 + cfg.n * cfg.s * 5, 1)}
    if cfg.hd:
        t = {f"fwht_pass{p}": (f"fwht_tile_kernel<{k}>", step.n_pad * cfg.d * 8, 1) for p, k in enumerate(step.plan)}
        t["gather"] = (gather_kernel_name(cfg), step.n_pad * cfg.d * 8 + cfg.m * cfg.d * 8 + step.n_pad * cfg.s * 5, 1)
        return t
    name = gather_kernel_name(cfg)
    return {"gather": (name, cfg.n * cfg.d * 8 + cfg.m * cfg.d * 8 + cfg.n * cfg.s * 5, 1)}


def gather_kernel_name(cfg):
    """The dense gather the library launches for this shape (csrc/gather.cu)."""
    if cfg.d % 2 == 0 and cfg.d > 64:
        return "gather_group_kernel<16>" if cfg.s > 1 else "gather_wide_kernel"
    return "gather_dense_kernel"


def traffic_record(cfg, layout):
    """ncu DRAM bytes (read + write) per launch of each kernel of this workload's
    step, from profiles/traffic.json (written from a committed launch list)."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(tp):
        return None
    with open(tp) as f:
        return json.load(f).get(f"{cfg.name}-{layout}")


def roofline(cfg, step, stage_ms, ms_step, peak_gbs, peak_src, layout="row", sketch="hashing"):
    """The dominant kernel against the HBM roofline, and the whole step's
    algorithmic-byte fraction, against the measured copy peak and
    the 8 TB/s spec."""
    table = kernel_table(cfg, step, layout, sketch)
    n_hash = getattr(step, "n_pad", cfg.n) if cfg.hd else cfg.n
    alg_step = alg_bytes_step(cfg, n_hash)
    present = {k: v for k, v in stage_ms.items() if k in table}
    name = max(present, key=lambda k: present[k])
    kern, alg, nl = table[name]
    t_launch = present[name] / nl
    achieved = alg / (t_launch / 1e3) / 1e9
    rec = traffic_record(cfg, layout)
    traffic = None
    step_traffic = None
    if rec:
        kt = rec.get("kernels", {})
        if name in kt:
            traffic = kt[name]["dram_bytes_per_launch"]
        if all(k in kt for k in present):
            step_traffic = sum(kt[k]["dram_bytes_per_launch"] * table[k][2] for k in present)
    ach_step = alg_step / (ms_step / 1e3) / 1e9
    per_kernel = {}
    for st, (kn, al, nl_) in table.items():
        if st not in present or present[st] <= 0:
            continue
        tl = present[st] / nl_
        a_ = al / (tl / 1e3) / 1e9
        tr = rec.get("kernels", {}).get(st, {}).get("dram_bytes_per_launch") if rec else None
        per_kernel[st] = {"kernel": kn, "ms_per_launch": round(tl, 4), "achieved": round(a_, 1),
                          "frac": round(a_ / peak_gbs, 4), "traffic": tr,
                          "dram_frac": (round(tr / (tl / 1e3) / 1e9 / peak_gbs, 4) if tr else None)}
    out = {"bound": "hbm", "kernel": kern, "stage": name, "achieved": round(achieved, 1), "peak": peak_gbs,
           "unit": "GB/s", "frac": round(achieved / peak_gbs, 4), "traffic": traffic,
           "alg_bytes_per_launch": alg, "ms_per_launch": round(t_launch, 4), "peak_source": peak_src,
           "frac_of_8tbs_spec": round(achieved / SPEC_HBM_GBS, 4),
           "dram_frac": (round(traffic / (t_launch / 1e3) / 1e9 / peak_gbs, 4) if traffic else None),
           "traffic_ratio": (round(traffic / alg, 3) if traffic else None),
           "traffic_source": rec.get("source") if rec else None,
           "step": {"alg_bytes": alg_step, "achieved": round(ach_step, 1), "alg_frac": round(ach_step / peak_gbs, 4),
                    "alg_frac_of_8tbs_spec": round(ach_step / SPEC_HBM_GBS, 4), "traffic": step_traffic,
                    "traffic_ratio": (round(step_traffic / alg_step, 3) if step_traffic else None),
                    "note": "SURVEY §8(d): |A| + |b| + |SA| + |Sb| + s*5 B of lists per hashed row, over the "
                            "step time"},
           "per_kernel": per_kernel}
    return out


def default_layout(cfg):
    """Storage of dense A the bench times by default: column-major (the paper's
    LAPACK/FFTW layout) for an H D workload whose row-major transform
    needs >= 3 HBM passes -- there the two-pass column-major plan (pass 2 fused
    with the sketch) moves 3|A| instead of 7|A| and wins (C5) -- or whose hash is
    s = 1 (C2: the column-major step, hash + tile lists beside pass 1, 0.44 ms vs
    0.50 row-major); else row-major (C3HD, s = 2: 3.69 vs 3.84 ms; plain
    sketches: one read)."""
    if not cfg.hd or cfg.kind == "csr":
        return "row"
    from paper_2105_11815_b200 import api
    n_pad = 1 << max(0, (cfg.n - 1).bit_length())
    return "col" if (len(api.rht_pass_plan(n_pad.bit_length() - 1, cfg.d)) >= 3 or cfg.s == 1) else "row"


def freivalds_check(cfg, SA, inputs, layout, nprobe=4):
    """Oracle-side whole-matrix check of the timed step's SA (SURVEY §8(c) tier
    2): w^T (S A) v vs (S^T w)^T (A v) with S^T w from the oracle's column lists
    (oracle/probes.py) and A v an fp64 library product of the input; bound
    1e-12 ||w|| ||SA||_F ||v||."""
    import numpy as np
    import torch

    from oracle import probes
    SA = SA.detach().cpu().numpy()
    if layout == "col" and cfg.kind != "csr":
        SA = SA.T
    if cfg.kind == "csr":
        import scipy.sparse as sp

        from synth import gen
        rp, ci, v = gen.csr(cfg)
        A = sp.csr_matrix((v, ci, rp), shape=(cfg.n, cfg.d))
        Av_of = lambda x: A @ x  # noqa: E731
    else:
        X = inputs[0]
        M = X.t() if layout == "col" else X
        Av_of = lambda x: torch.mv(M, torch.from_numpy(x).to(M.device)).cpu().numpy()  # noqa: E731
    rng = np.random.default_rng(2105)
    worst = 0.0
    for _ in range(nprobe):
        w, v = rng.standard_normal(cfg.m), rng.standard_normal(cfg.d)
        lhs = float(w @ (SA @ v))
        rhs = (probes.probe_rht if cfg.hd else probes.probe_dense)(cfg.seed, cfg.n, cfg.m, cfg.s, w, Av_of(v))
        worst = max(worst, abs(lhs - rhs) / (np.linalg.norm(w) * np.linalg.norm(SA) * np.linalg.norm(v)))
    return {"ok": bool(worst <= 1e-12), "worst_rel": worst, "probes": nprobe, "bound": 1e-12,
            "what": "w^T(SA)v vs (S^T w)^T(Av): all m x d entries of SA, oracle column lists"}


def capture_step(step, torch):
    """Capture one step.run() into a CUDA graph (the step's kernels, side-stream
    fork/join included; nothing is cached: every replay redraws S and recomputes
    SA, Sb).  Returns (graph, kernels per step)."""
    import paper_2105_11815_b200 as skh
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step.run()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    n0 = skh.api.launch_count()
    with torch.cuda.graph(g, capture_error_mode="thread_local"):
        step.run()
    per_step = skh.api.launch_count() - n0
    g.replay()
    torch.cuda.synchronize()
    return g, per_step


GRAPH_MAX_MS = 2.0  # longer steps gain nothing from a graph (C5: 15 launches in 45 ms; C3HD 3.7 ms:
#                     its side-stream branch replayed 3.75 vs 3.65-3.69 ms eager)


def time_step(step, steps, torch, graph=True):
    """K timed steps.  Stage times come from an eager pass of K steps with CUDA
    events after every stage (on the launching streams); the step time is then
    taken over K replays of the step captured as one CUDA graph (launch
    overhead off the critical path: C1 0.067 -> 0.027 ms, C4 0.72 -> 0.68 ms),
    or from the eager pass itself with graph=False or a step longer than
    GRAPH_MAX_MS (not launch-bound).  Returns (ms per step,
    stage ms, kernels launched in the timed region, mode, eager ms per step)."""
    import paper_2105_11815_b200 as skh
    timers = [step.new_timer() for _ in range(steps)]
    torch.cuda.synchronize()
    n0 = skh.api.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(steps):
        step.run(timers[k])
    e1.record()
    torch.cuda.synchronize()
    launches = skh.api.launch_count() - n0
    ms_eager = e0.elapsed_time(e1) / steps
    per = [t.durations_ms() for t in timers]
    stage_ms = {k: sum(p[k] for p in per) / len(per) for k in per[0]}
    if not graph or ms_eager > GRAPH_MAX_MS:
        return ms_eager, stage_ms, launches, "eager", ms_eager
    try:
        g, per_step = capture_step(step, torch)
    except RuntimeError as e:  # a step that cannot be captured is timed eagerly
        torch.cuda.synchronize()
        return ms_eager, stage_ms, launches, f"eager (graph capture failed: {str(e)[:80]})", ms_eager
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del g
    return ms, stage_ms, per_step * steps, "cuda_graph", ms_eager


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
    clk = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
    clk.start()
    time.sleep(0.3)
    ms, stage_ms, launches, mode, ms_eager = time_step(step, args.steps, torch, not args.no_graph)
    clocks = clk.stop()
    pk, src = peaks()
    value = cfg.a_bytes / (ms / 1e3) / 1e9
    line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "pct_hbm_peak": round(100 * value / pk["hbm_gbs"], 2),
            "config": {"workload": cfg.name, "n": cfg.n, "d": cfg.d, "m": cfg.m, "s": cfg.s, "hd": cfg.hd,
                       "a_bytes": cfg.a_bytes, "layout": "column-major" if args.layout == "col" else "row-major",
                       "l2": "inputs (A) larger than L2; no flush",
                       "parallelism": "single GPU", "launch": mode, "note": cfg.note},
            "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()}, "ms_per_step_eager": round(ms_eager, 4),
            "gpu_launches": int(launches), "clocks": clocks}
    line["roofline"] = roofline(cfg, step, stage_ms, ms, pk["hbm_gbs"], src, args.layout, args.sketch)
    line["alg_frac"] = line["roofline"]["step"]["alg_frac"]
    SA_last = step.run()[0] if not args.no_cpu_baseline else None
    torch.cuda.synchronize()
    if args.sketch != "hashing":
        line["config"]["sketch"] = {"variant": "s-hashing variant (Def. 7)", "dht": "HR-DHT S_h F D (eq. (6.1))",
                                    "srdht": "SR-DHT S_s F D (eq. (7.2))"}[args.sketch]
    if SA_last is not None and args.sketch == "hashing":
        # the oracle leg: a whole-matrix Freivalds check of the timed object's SA
        fv = freivalds_check(cfg, SA_last, inputs, args.layout)
        line["freivalds_ok"] = fv["ok"]
        cpu_line = dict(cpu_line or {}, freivalds=fv)
    del step, SA_last
    if not args.no_e2e:
        line["e2e"] = e2e_measure(cfg, inputs, args.e2e_steps, torch, args.layout) if args.sketch == "hashing" else None
    del inputs
    torch.cuda.empty_cache()
    if cfg.kind != "csr" and cfg.hd and args.sketch == "hashing" and not args.no_alt_layout:
        alt = "row" if args.layout == "col" else "col"
        line["row_major" if alt == "row" else "column_major"] = alt_layout_measure(args, cfg, torch, pk, src, alt)
        torch.cuda.empty_cache()
    if cpu_line is not None:
        line["cpu_baseline"] = cpu_line
    if args.sketch == "hashing" and not args.no_all_workloads:
        line["workloads"] = other_workloads_measure(args, cfg, torch, pk, src)
        line["next_rows"] = next_rows_measure(args, torch, pk)
    print(json.dumps(line), flush=True)


def other_workloads_measure(args, main_cfg, torch, pk, src):
    """The other BASELINE configs in the same run (so the driver's clock covers
    them too): each in its default layout, W warm-up + min(K, 10) timed steps,
    the step's SURVEY §8(d) alg_frac and a whole-matrix Freivalds check of its
    SA (the oracle leg).  Reported beside the headline, not instead of it."""
    from synth import configs
    out = {}
    for name in ("C1", "C2", "C3", "C3HD", "C4", "C5"):
        cfg = configs.ALL[name]
        if name == main_cfg.name:
            continue
        layout = default_layout(cfg)
        step, inputs = build_step(cfg, torch, layout)
        torch.cuda.synchronize()
        for _ in range(max(args.warmup, 0)):
            step.run()
        steps = max(1, min(args.steps, 10))
        ms, stage_ms, _, mode, ms_eager = time_step(step, steps, torch, not args.no_graph)
        rl = roofline(cfg, step, stage_ms, ms, pk["hbm_gbs"], src, layout)
        rec = {"value": round(cfg.a_bytes / (ms / 1e3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
               "steps": steps, "layout": "column-major" if layout == "col" else "row-major", "launch": mode,
               "ms_per_step_eager": round(ms_eager, 4),
               "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
               "alg_frac": rl["step"]["alg_frac"], "kernel": rl["kernel"], "kernel_frac": rl["frac"]}
        if not args.no_cpu_baseline:
            SA = step.run()[0]
            torch.cuda.synchronize()
            fv = freivalds_check(cfg, SA, inputs, layout)
            rec["freivalds_ok"], rec["freivalds_worst_rel"] = fv["ok"], fv["worst_rel"]
            del SA
        out[name] = rec
        del step, inputs
        torch.cuda.empty_cache()
    return out


def next_rows_measure(args, torch, pk):
    """SURVEY §8(f) "next" rows on C2 in the same run (driver-measured): NEXT-1
    Algorithm 1 Steps 2-5 (the paper's default rank-revealing Step 2, rcond
    1e-12, then LSQR to the (7.1) stop) on the timed step's SA, Sb; NEXT-2 the
    s-hashing variant sketch; NEXT-3 HR-DHT and NEXT-4 SR-DHT sketches.  Each
    sketch: W warm-up + min(K, 10) timed steps (CUDA-graph replays, as above);
    the solve: one warm-up and one timed call with the library's stage trace."""
    import paper_2105_11815_b200 as skh
    from synth import configs
    cfg = configs.ALL["C2"]
    out = {"workload": cfg.name}
    steps = max(1, min(args.steps, 10))
    for key, sk in (("next2_variant", "variant"), ("next3_hrdht", "dht"), ("next4_srdht", "srdht")):
        step, inputs = build_step(cfg, torch, "row", sk)
        for _ in range(max(args.warmup, 0)):
            step.run()
        ms, stage_ms, _, mode, ms_eager = time_step(step, steps, torch, not args.no_graph)
        out[key] = {"ms_per_step": round(ms, 4), "launch": mode, "ms_per_step_eager": round(ms_eager, 4),
                    "value": round(cfg.a_bytes / (ms / 1e3) / 1e9, 2), "unit": "GB/s",
                    "alg_frac": round(alg_bytes_step(cfg, cfg.n) / (ms / 1e3) / 1e9 / pk["hbm_gbs"], 4),
                    "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()}}
        del step, inputs
        torch.cuda.empty_cache()
    step, (A, b) = build_step(cfg, torch, "row")
    SA, Sb = step.run()
    SA, Sb = SA.clone(), Sb.clone()
    del step
    solver = skh.LlsSolver(cfg.n, cfg.d, cfg.m, rcond=1e-12)
    solver(A, b, SA, Sb)  # warm-up: handles, cuSOLVER workspace
    torch.cuda.synchronize()
    with skh.Trace(16) as tr:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, info = solver(A, b, SA, Sb)
        e1.record()
    torch.cuda.synchronize()
    st = tr.durations_ms()
    it = max(info["iters"], 1)
    per_it = st.get("lsqr", 0.0) / it
    gbs = 2 * cfg.a_bytes / (per_it / 1e3) / 1e9 if per_it > 0 else None
    out["next1_solve"] = {"ms": round(e0.elapsed_time(e1), 3), "step2": "rank-revealing (rcond 1e-12)",
                          "rank": info["rank"], "iters": info["iters"], "stop_test2": info["test2"],
                          "exit_step": info["step"], "stages_ms": {k: round(v, 3) for k, v in st.items()},
                          "ms_per_lsqr_iter": round(per_it, 4),
                          "lsqr_A_frac": (round(gbs / pk["hbm_gbs"], 3) if gbs else None),
                          "note": "each LSQR iteration reads A twice (A R^-1 v, A^T u)"}
    del A, b, SA, Sb, x, solver
    torch.cuda.empty_cache()
    return out


def alt_layout_measure(args, cfg, torch, pk, src, layout):
    """The same workload stored in the other layout, timed the same way and
    reported beside the headline (column-major: skh_rht_dense_colmajor's two
    passes; row-major: the tile passes + gather, §5)."""
    step, inputs = build_step(cfg, torch, layout)
    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 0)):
        step.run()
    ms, stage_ms, _, mode, _ = time_step(step, args.steps, torch, not args.no_graph)
    out = {"value": round(cfg.a_bytes / (ms / 1e3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(ms, 4),
           "launch": mode,
           "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
           "roofline": roofline(cfg, step, stage_ms, ms, pk["hbm_gbs"], src, layout),
           "note": ("same A stored column-major; pass 1 (13 contiguous bits, D fused) + pass 2 fused with the "
                    "gather: 3|A| of HBM traffic; SA to 1e-12 (DESIGN.md R17)" if layout == "col" else
                    "same A stored row-major; tile FWHT passes + gather: (2 passes + 1)|A| of HBM traffic; "
                    "SA bit-identical to the oracle")}
    del step, inputs
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--layout", default="auto", choices=["auto", "row", "col"],
                    help="storage of dense A: row-major, column-major (the paper's LAPACK layout), or auto "
                         "(default_layout: column-major for H D workloads whose row-major plan needs >= 3 passes)")
    ap.add_argument("--impl", default="skh", choices=["skh", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--sketch", default="hashing", choices=["hashing", "variant", "dht", "srdht"],
                    help="hashing (default, Def. 4 / HRHT), the s-hashing variant (Def. 7), HR-DHT (eq. 6.1) "
                         "or SR-DHT (eq. 7.2)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt-layout", action="store_true",
                    help="skip the column-major measurement reported beside a row-major H D workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the K steps as eager launches instead of K replays of the step's CUDA graph")
    ap.add_argument("--no-all-workloads", action="store_true",
                    help="skip the other BASELINE configs reported beside the headline (line key 'workloads')")
    args = ap.parse_args()
    from synth import configs
    cfg = configs.ALL[args.workload]
    if args.impl == "reference":
        return reference_arm(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        if args.layout == "col":
            raise SystemExit("--layout col is single-GPU in this build (sharded runs use row-major A)")
        from paper_2105_11815_b200 import sharded_bench
        return sharded_bench.run(args, cfg)
    from paper_2105_11815_b200 import build
    build.build()
    if args.layout == "auto":
        args.layout = default_layout(cfg)
    return gpu_arm_single(args, cfg)


def self_launch(args):
    """`python bench.py --gpus N` without a launcher: start N ranks with
    torch.distributed.run on this node (127.0.0.1) and pass their output
    through; rank 0 prints the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()
