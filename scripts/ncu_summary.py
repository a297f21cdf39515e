"""Summarise an ncu --set full capture (.ncu-rep) into a small markdown /
json pair under profiles/ (or OUTDIR).  Usage: python scripts/ncu_summary.py REP NAME [OUTDIR]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main(rep, name, outdir="profiles"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    out = {k: d.get(k) for k in KEYS}
    out["kernel"] = d.get("Kernel Name")
    stalls = {k.split("issue_stalled_")[1].split("_per_issue")[0]: float(d[k])
              for k in h if k.startswith("smsp__average_warps_issue_stalled") and d.get(k)
              and float(d[k]) > 0.1}
    out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
    rd = float(d["dram__bytes_read.sum"]) * (1e6 if u.get("dram__bytes_read.sum") == "Mbyte" else 1)
    wr = float(d["dram__bytes_write.sum"]) * (1e6 if u.get("dram__bytes_write.sum") == "Mbyte" else 1)
    out["bytes_per_launch"] = rd + wr
    json.dump(out, open(f"{outdir}/{name}.json", "w"), indent=1)
    with open(f"{outdir}/{name}.md", "w") as f:
        f.write(f"# {name}: ncu --set full summary\n\nkernel: `{out['kernel']}`\n\n")
        for k in KEYS:
            f.write(f"- {k} = {d.get(k)} {u.get(k, '')}\n")
        f.write(f"- dram read+write bytes per launch = {rd + wr:.0f}\n")
        f.write("\nstall reasons (warps per issue):\n\n")
        for k, val in out["stalls_per_issue"].items():
            f.write(f"- {k}: {val:.2f}\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
