"""Write profiles/traffic.json (ncu DRAM bytes per launch of each bench stage)
from the committed launch lists (tools/launch_lists.sh output):
   python tools/traffic_from_launches.py profiles/r02/launches"""
import csv
import io
import json
import os
import sys

# bench stage -> kernels it launches (name prefixes; summed per launch of the stage)
STAGES = {
    "C5-col": {"pass1": ["cm_pass1"], "pass2_gather": ["cm_gather_kernel"]},
    "C5-row": {"fwht_pass0": ["fwht_tile_kernel<7, 1>"], "fwht_pass1": ["fwht_tile_kernel<7, 0>"],
               "fwht_pass2": ["fwht_tile_kernel<7, 0>"], "gather": ["gather_wide_kernel"]},
    "C2-col": {"pass1": ["cm_pass1"], "pass2_gather": ["cm_gather_kernel"]},
    "C2-row": {"fwht_pass0": ["fwht_tile_kernel<8, 1>"], "fwht_pass1": ["fwht_tile_kernel<8, 0>"],
               "gather": ["gather_wide_kernel"]},
    "C3HD-row": {"fwht_pass0": ["fwht_tile_kernel<9, 1>"], "fwht_pass1": ["fwht_tile_kernel<8, 0>"],
                 "gather": ["gather_group_kernel"]},
    "C3-row": {"gather": ["gather_group_kernel"]},
    "C4-row": {"gather_csr": ["csr_len_kernel", "csr_expand_kernel", "csr_reduce_kernel"]},
    "C1-row": {"gather": ["gather_dense_kernel"]},
}
FILES = {"C5-col": "C5_auto", "C5-row": "C5_row", "C2-col": "C2_auto", "C2-row": "C2_row", "C3HD-row": "C3HD_auto",
         "C3-row": "C3_auto", "C4-row": "C4_auto", "C1-row": "C1_auto"}


def launches(path):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    per = {}
    for r in rows:
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return list(per.values())


def main(src):
    out = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of each bench stage's kernels, mean "
                    "over the launch list of `python bench.py --workload W --layout L --steps 2 --warmup 1 --no-e2e "
                    "--no-cpu-baseline --no-alt-layout` under ncu --clock-control none (tools/launch_lists.sh); "
                    "bench.py copies the matching entries into roofline.traffic / roofline.step.traffic."}
    for key, stages in STAGES.items():
        path = os.path.join(src, f"launches_{FILES[key]}.csv")
        if not os.path.exists(path):
            continue
        ls = launches(path)
        kt = {}
        for st, prefixes in stages.items():
            tot, n = 0.0, 0
            for p in prefixes:
                sel = [x for x in ls if p in x["name"].replace("(anonymous namespace)::", "")]
                if not sel:
                    continue
                tot += sum(x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in sel) / len(sel)
                n += 1
            if n:
                kt[st] = {"dram_bytes_per_launch": int(tot), "kernels": prefixes}
        out[key] = {"kernels": kt, "source": path}
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json"),
              "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:2000])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02/launches")
