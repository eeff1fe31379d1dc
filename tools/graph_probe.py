"""Eager vs CUDA-graph replay of the bench step objects (one GPU): captures
step.run() once into a torch.cuda.CUDAGraph and times K replays against K eager
calls, CUDA events on the current stream.  Also checks that the replayed SA is
bit-identical to the eager one.

    python tools/graph_probe.py [C1 C2 ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from synth import configs  # noqa: E402


def timeit(fn, k):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def main():
    names = sys.argv[1:] or ["C1", "C2", "C3", "C3HD", "C4"]
    torch.cuda.set_device(0)
    for name in names:
        cfg = configs.ALL[name]
        layout = bench.default_layout(cfg)
        step, inputs = bench.build_step(cfg, torch, layout)
        for _ in range(3):
            step.run()
        k = 50 if cfg.a_bytes < (1 << 31) else 10
        t_eager = timeit(step.run, k)
        ref = [x.clone() if x is not None else None for x in step.run()]
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step.run()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            out = step.run()
        g.replay()
        torch.cuda.synchronize()
        same = all((a is None and b is None) or torch.equal(a, b) for a, b in zip(ref, out))
        t_graph = timeit(g.replay, k)
        print(f"{name} {layout}: eager {t_eager:.4f} ms, graph {t_graph:.4f} ms, bit-identical {same}", flush=True)
        del g, step, inputs, out, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
