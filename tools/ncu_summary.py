"""Summarise `ncu --set full` reports into the JSON kept under profiles/.

usage: python tools/ncu_summary.py OUT.json REPORT.ncu-rep [REPORT2.ncu-rep ...]

Per captured kernel launch (first launch of each kernel name wins): duration,
DRAM bytes, DRAM / SM / FP64-pipe utilisation, occupancy, registers, L2 read
sectors and the top warp-stall reasons -- the numbers DESIGN.md and
profiles/README.md quote.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0]
        if name in out:
            continue
        rec = {}
        for m in METRICS:
            if m in d:
                rec[m] = f"{d[m]} {u.get(m, '')}".strip()
        stalls = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k] or 0))
                  for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued")]
        tot = sum(v for _, v in stalls) or 1.0
        rec["top_stalls_pct"] = {k: round(100 * v / tot, 1)
                                 for k, v in sorted(stalls, key=lambda x: -x[1])[:5]}
        rec["report"] = path.split("/")[-1]
        out[name] = rec
    return out


def main():
    out_path, reports = sys.argv[1], sys.argv[2:]
    res = {}
    for r in reports:
        res.update(summarise(r))
    with open(out_path, "w") as fh:
        json.dump(res, fh, indent=1)
    for k, v in res.items():
        print(f"{k:40s} {v.get('gpu__time_duration.sum', '')}")


if __name__ == "__main__":
    main()
