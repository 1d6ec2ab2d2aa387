"""Summarise ncu captures (.ncu-rep, --set full) into profiles/ (markdown + JSON).

    python tools/ncu_summary.py gpurun_out/prof_ndft.ncu-rep [...] --out profiles/round1

Writes <out>_kernels.md (human summary) and <out>_kernels.json (per-kernel
metrics; bench.py reads dram bytes per launch from it for roofline.traffic).
"""

import argparse
import csv
import io
import json
import re
import subprocess

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_pct": "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "dram_gbs": "dram__bytes.sum.per_second",
    "warps_active_per_sched": "smsp__warps_active.avg.per_cycle_active",
    "inst_executed": "smsp__inst_executed.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
}
UNIT_SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "byte": 1.0,
              "ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3,
              "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "second": 1e3,
              "Gbyte/s": 1.0, "Tbyte/s": 1e3, "Mbyte/s": 1e-3}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")[:160]}
        for name, m in KEYS.items():
            v = d.get(m)
            if v in (None, ""):
                continue
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                continue
            f *= UNIT_SCALE.get(u.get(m, ""), 1.0)
            k[name] = f
        st = {}
        for m, v in d.items():
            mm = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active\.ratio$", m)
            if mm and v:
                st[mm.group(1)] = round(float(v), 3)
        k["stalls_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:8])
        kernels.append(k)
    return kernels


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    allk = {}
    md = ["| kernel | ms | DRAM rd+wr (MB) | issue % | FMA pipe % | ALU pipe % | DRAM % | regs | top stalls |",
          "|---|---|---|---|---|---|---|---|---|"]
    for rep in a.reps:
        for k in load(rep):
            name = re.sub(r"\(.*", "", k["kernel"]).replace("void ", "").replace("<unnamed>::", "")
            allk[name + " @" + rep.split("/")[-1]] = k
            tr = (k.get("dram_read_bytes", 0) + k.get("dram_write_bytes", 0)) / 1e6
            stalls = ", ".join(f"{s}={v}" for s, v in list(k["stalls_per_issue"].items())[:4])
            md.append(f"| {name} | {k.get('duration_ms', 0):.3f} | {tr:.1f} | {k.get('issue_active_pct', 0):.1f} | "
                      f"{k.get('fma_pipe_pct', 0):.1f} | {k.get('alu_pipe_pct', 0):.1f} | {k.get('dram_pct', 0):.1f} | "
                      f"{int(k.get('registers', 0))} | {stalls} |")
    with open(a.out + "_kernels.json", "w") as f:
        json.dump(allk, f, indent=1)
    with open(a.out + "_kernels.md", "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
