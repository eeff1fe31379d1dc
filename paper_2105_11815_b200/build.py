"""Build the in-tree shared libraries with nvcc for sm_100a.

  libskh.so   (paper_2105_11815_b200/csrc/*.cu)  -- the product: C ABI of include/skh.h
  libsynth.so (synth/csrc/*.cu)                  -- device input generator (harness)

Usage: python -m paper_2105_11815_b200.build [--force]
"""
import concurrent.futures
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2105_11815_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
# SKH_CHECKED=1: the checked build (device-side SKH_CHECK invariants, common.cuh);
# always a full rebuild, and the next plain build rebuilds again
CHECKED = os.environ.get("SKH_CHECKED", "0") == "1"
if CHECKED:
    FLAGS = FLAGS + ["-DSKH_CHECKED"]

TARGETS = {
    os.path.join(PKG, "libskh.so"): sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu"))),
    os.path.join(ROOT, "synth", "libsynth.so"): sorted(glob.glob(os.path.join(ROOT, "synth", "csrc", "*.cu"))),
}
# extra link libraries: the LLS solve (csrc/lls.cu, Alg. 1 Steps 2-5) calls
# cuSOLVER dgeqrf/dormqr and cuBLAS dtrsv for the small d x d factor work; the
# HR-DHT sketch (csrc/dht.cu) calls cuFFT for the Hartley transform
LIBS = {os.path.join(PKG, "libskh.so"): ["-lcusolver", "-lcublas", "-lcufft"]}


def _deps(srcs):
    d = list(srcs)
    for s in srcs:
        d += glob.glob(os.path.join(os.path.dirname(s), "*.cuh"))
    d += [os.path.join(ROOT, "include", "skh.h")]
    return d


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in _deps(srcs) if os.path.exists(s))


def _compile(src, obj, verbose):
    cmd = [NVCC, *ARCH, *FLAGS, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {src}")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(force=False, verbose=False):
    """Compile stale objects (in parallel) and relink stale libraries."""
    built = []
    for out, srcs in TARGETS.items():
        if not srcs:
            continue
        stamp = out + ".checked"
        was_checked = os.path.exists(stamp)
        if not force and not _stale(out, srcs) and was_checked == CHECKED:
            continue
        force = force or was_checked != CHECKED
        objdir = os.path.join(os.path.dirname(out), "build_obj")
        os.makedirs(objdir, exist_ok=True)
        objs = [os.path.join(objdir, os.path.basename(s).replace(".cu", ".o")) for s in srcs]
        todo = [(s, o) for s, o in zip(srcs, objs) if force or _stale(o, [s])]
        with concurrent.futures.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
            for f in [ex.submit(_compile, s, o, verbose) for s, o in todo]:
                f.result()
        cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcudart", *LIBS.get(out, [])]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"link failed for {out}")
        if CHECKED:
            open(stamp, "w").close()
        elif os.path.exists(stamp):
            os.remove(stamp)
        built.append(out)
    return built


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
