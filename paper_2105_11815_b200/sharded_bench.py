"""bench.py's multi-GPU arm (torchrun, one process per GPU).

Strong scaling of the BASELINE workload over N ranks (C5: "row-sharded over 8
GPUs; runs at 1/2/4/8 GPUs"): rank r holds rows [r n/N, (r+1) n/N) of A and
runs the sharded step of sharded.py (local FWHT passes, one all-to-all of rows,
the cross stages, hash of its rows, gather, all-to-all of SA strips + rank-order
sum).  Timed with CUDA events on every rank between barriers, reported as the
max over ranks; rank 0 prints the JSON line.  The collectives use NCCL over
NVLink/NVSwitch; SKH_DIST_BACKEND=gloo runs the same path functionally (host-
staged collectives) for single-GPU smoke tests.
"""
import json
import os
import time


def _stage_events(names, torch):
    evs = {"start": torch.cuda.Event(enable_timing=True)}
    for n in names:
        evs[n] = torch.cuda.Event(enable_timing=True)
    return evs


def comm_sweep(torch, dist, backend, sizes, iters=5):
    """In-run collective roofline: all_to_all_single and
    reduce_scatter_tensor at the message sizes the sharded step uses (bytes per
    rank), timed with CUDA events on every rank (max over ranks).  Bus
    bandwidth = bytes per rank x (G-1)/G / time, NCCL's convention for both."""
    G = dist.get_world_size()
    dev = torch.device("cuda", torch.cuda.current_device())
    out = []
    for op, nbytes in sizes:
        n = max(G, (int(nbytes) // 8) // G * G)
        x = torch.randn(n, dtype=torch.float64, device=dev)
        y = torch.empty(n if op == "all_to_all" else n // G, dtype=torch.float64, device=dev)
        if backend == "gloo":
            x, y = x.cpu(), y.cpu()

        def once():
            if op == "all_to_all":
                dist.all_to_all_single(y, x)
            else:
                dist.reduce_scatter_tensor(y, x) if backend != "gloo" else dist.all_reduce(x)
        for _ in range(2):
            once()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            once()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64,
                         device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        bus = n * 8 * (G - 1) / G / (ms / 1e3) / 1e9
        out.append({"op": op if backend != "gloo" or op == "all_to_all" else "all_reduce (gloo)",
                    "bytes_per_rank": n * 8, "ms": round(ms, 4), "busbw_GBps": round(bus, 1)})
    return out


def run(args, cfg):
    import torch
    import torch.distributed as dist

    from . import api, build, sharded
    from synth import device

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("SKH_DIST_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    dev = local % max(ndev, 1)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)
    G = dist.get_world_size()
    if rank == 0:
        build.build()
    dist.barrier()

    def red_max(x):
        t = torch.tensor([float(x)], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def red_sum(x):
        t = torch.tensor([float(x)], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- inputs (this rank's shard) and the sharded step
    if cfg.kind == "csr":
        rp, ci, v = device.csr(cfg)
        b = device.rhs(cfg)
        step = sharded.ShardedCsr(cfg.seed, rp, ci, v, cfg.d, b, cfg.m, cfg.s)
        shard = None
    elif cfg.hd:
        L = cfg.n // G
        b = device.rhs(cfg, rank * L, (rank + 1) * L)
        # SKH_SHARDED_HD: m2 (butterfly all-to-all), m3 (exchange-free, row-major
        # pull gather), m3col (exchange-free, column-major, on-chip fan-out);
        # auto = m3col at G = 2 (projected 0.78 vs 0.70 strong-scaling
        # efficiency from the measured per-rank kernels), else m2
        mode = os.environ.get("SKH_SHARDED_HD", "auto")
        if mode == "auto":
            mode = "m3col" if (G == 2 and G * cfg.s <= 8) else "m2"
        if mode == "m3col":
            A = device.dense_colmajor(cfg, rank * L, (rank + 1) * L)
            step = sharded.ShardedHrhtM3Col(cfg.seed, A, b, cfg.n, cfg.m, cfg.s)
        else:
            A = device.dense(cfg, rank * L, (rank + 1) * L)
            if mode == "m3":
                step = sharded.ShardedHrhtM3(cfg.seed, A, b, cfg.n, cfg.m, cfg.s)
            else:
                step = sharded.ShardedHrht(cfg.seed, A, b, cfg.n, cfg.m, cfg.s)
        shard = (A, b)
    else:
        per = (cfg.n + G - 1) // G
        r0, r1 = min(cfg.n, rank * per), min(cfg.n, (rank + 1) * per)
        A = device.dense(cfg, r0, r1)
        b = device.rhs(cfg, r0, r1)
        step = sharded.ShardedPlain(cfg.seed, A, b, cfg.n, cfg.m, cfg.s)
        shard = (A, b)
    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 0)):
        step.run()
    torch.cuda.synchronize()

    # ---- timed region
    names = list(step.STAGES)
    evsets = [_stage_events(names, torch) for _ in range(args.steps)]
    clk = None
    if rank == 0:
        from bench import ClockSampler
        clk = ClockSampler(dev)
        clk.start()
        time.sleep(0.3)
    n0 = api.launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.steps):
        evs = evsets[k]
        evs["start"].record()
        step.run(mark=lambda nm, evs=evs: evs[nm].record())
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    launches = red_sum(api.launch_count() - n0)
    clocks = clk.stop() if clk else None
    ms = red_max(e0.elapsed_time(e1)) / args.steps
    stage_ms = {}
    for nm in names:
        tot = 0.0
        for evs in evsets:
            prev = "start" if nm == names[0] else names[names.index(nm) - 1]
            tot += evs[prev].elapsed_time(evs[nm])
        stage_ms[nm] = red_max(tot / len(evsets))

    # ---- e2e: the same step fed from this rank's pinned host shard, strip read back
    e2e = None
    if shard is not None and not args.no_e2e:
        A_d, b_d = shard
        A_h = torch.empty(A_d.shape, dtype=torch.float64, pin_memory=True)
        A_h.copy_(A_d)
        b_h = torch.empty(b_d.shape, dtype=torch.float64, pin_memory=True)
        b_h.copy_(b_d)
        torch.cuda.synchronize()
        t = []
        out_bytes = 0
        for _ in range(args.e2e_steps):
            dist.barrier()
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            A_d.copy_(A_h, non_blocking=True)
            b_d.copy_(b_h, non_blocking=True)
            res = step.run()
            SA, Sb = res[0], res[2] if len(res) == 4 else res[1]
            SA_h = SA.cpu()
            Sb_h = Sb.cpu()
            s1.record()
            torch.cuda.synchronize()
            out_bytes = SA_h.numel() * 8 + Sb_h.numel() * 8
            t.append(s0.elapsed_time(s1))
        ms_e2e = red_max(sum(t) / len(t))
        e2e = {"value": cfg.a_bytes / (ms_e2e / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms_e2e,
               "steps": args.e2e_steps, "h2d_bytes_per_step": int(red_sum(A_h.numel() * 8 + b_h.numel() * 8)),
               "d2h_bytes_per_step": int(red_sum(out_bytes)), "api": type(step).__name__ + ".run (pinned shard)"}

    # ---- collective roofline at the step's message sizes (all ranks take part)
    msg = []
    if cfg.hd and G > 1 and isinstance(step, sharded.ShardedHrht):
        # one column chunk of the butterfly exchange: the L x W send buffer of a rank
        msg.append(("all_to_all", (cfg.n // G) * min(cfg.d, getattr(step, "W", cfg.d)) * 8))
    if G > 1 and cfg.kind != "csr":
        msg.append(("reduce_scatter", ((cfg.m + G - 1) // G) * G * cfg.d * 8))
    sweep = comm_sweep(torch, dist, backend, msg) if msg else []

    if rank == 0:
        from bench import METRIC, peaks
        pk, src = peaks()
        value = cfg.a_bytes / (ms / 1e3) / 1e9
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": G, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "pct_hbm_peak": round(100 * value / (G * pk["hbm_gbs"]), 2),
                "config": {"workload": cfg.name, "n": cfg.n, "d": cfg.d, "m": cfg.m, "s": cfg.s, "hd": cfg.hd,
                           "a_bytes": cfg.a_bytes, "l2": "inputs (A) larger than L2; no flush",
                           "parallelism": f"row-sharded x{G} ({type(step).__name__}, {backend})",
                           "note": cfg.note},
                "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
                "gpu_launches": int(launches), "clocks": clocks, "e2e": e2e}
        if cfg.hd and isinstance(step, sharded.ShardedHrhtM3Col):
            # per rank: pass 1 of H_L D A_r and the fused pass 2, whose gather adds
            # every local row (read once) into its G s folded buckets on chip --
            # SURVEY §8(d) counts A_r once, the partial SA^T and the folded lists
            L = cfg.n // G
            t = stage_ms["sketch"]
            alg = L * cfg.d * 8 + cfg.m * cfg.d * 8 + G * cfg.s * L * 5
            ach = alg / (t / 1e3) / 1e9
            line["roofline"] = {"bound": "hbm", "kernel": "cm_pass1p + cm_gather (G s folded draws per row) per rank",
                                "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                                "frac": round(ach / pk["hbm_gbs"], 4), "traffic": None, "peak_source": src,
                                "sketch_ms": round(t, 4), "draws_per_local_row": G * cfg.s}
            dq = (cfg.d + G - 1) // G
            line["comm"] = {"all_to_all_rows_bytes_sent_per_rank": 0,
                            "strip_reduction_bytes_per_rank": (G - 1) * dq * cfg.m * 8}
        elif cfg.hd and isinstance(step, sharded.ShardedHrhtM3):
            # per rank: the local FWHT passes over L rows, then a gather whose lists
            # read every local row G s times (the folded H_G)
            L = cfg.n // G
            npass = len(api.rht_pass_plan((L).bit_length() - 1, cfg.d))
            t = stage_ms["transform"] + stage_ms["gather"]
            # per rank: the local passes read Z_r once each (d 8 B per
            # row per launch), the gather reads every local row G s times (the
            # folded H_G) and writes the partial m x d
            alg = npass * L * cfg.d * 8 + G * cfg.s * L * cfg.d * 8 + cfg.m * cfg.d * 8
            ach = alg / (t / 1e3) / 1e9
            line["roofline"] = {"bound": "hbm", "kernel": f"local FWHT passes ({npass}) + folded gather per rank",
                                "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                                "frac": round(ach / pk["hbm_gbs"], 4), "traffic": None, "peak_source": src,
                                "gather_ms": round(stage_ms["gather"], 4),
                                "gather_row_reads_per_local_row": G * cfg.s,
                                "gather_read_bytes_per_rank": G * cfg.s * L * cfg.d * 8}
            line["comm"] = {"all_to_all_rows_bytes_sent_per_rank": 0,
                            "strip_reduction_bytes_per_rank": (G - 1) * ((cfg.m + G - 1) // G) * cfg.d * 8}
        elif cfg.hd:
            # the column-chunk pipeline interleaves the kernels with the (overlapped)
            # all-to-all, so the roofline is taken over the whole pipeline stage:
            # algorithmic HBM bytes of the local passes, the cross-stage pass and
            # the gather, per rank, over the stage's time
            L = cfg.n // G
            npass = len(api.rht_pass_plan((L).bit_length() - 1, min(cfg.d, step.W)))
            ncross = 1 if G > 1 else 0
            alg = (npass + ncross) * 2 * L * cfg.d * 8 + L * cfg.d * 8 + cfg.m * cfg.d * 8
            t = stage_ms["pipeline"]
            ach = alg / (t / 1e3) / 1e9
            line["roofline"] = {"bound": "hbm", "kernel": f"pipeline per rank ({npass} local FWHT passes + "
                                f"{ncross} cross pass + gather, {step.K} column chunks of {step.W})",
                                "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                                "frac": round(ach / pk["hbm_gbs"], 4), "traffic": None, "peak_source": src}
            a2a_bytes = (G - 1) * (L // G) * cfg.d * 8
            line["comm"] = {"all_to_all_rows_bytes_sent_per_rank": a2a_bytes,
                            "overlapped_with": "compute of the neighbouring column chunks",
                            "pipeline_ms": round(t, 4), "peer_peak_GBps": 770.0,
                            "peak_source": "B200_PROFILING.md measured peer copy"}
        line.setdefault("comm", {})["measured"] = sweep
        line["comm"]["backend"] = backend
        if backend != "nccl":
            line["comm"]["note"] = "gloo: host-staged collectives (functional run), not NVLink"
        line["comm"].pop("peer_peak_GBps", None)
        line["comm"].pop("peak_source", None)
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
