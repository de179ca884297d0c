"""Summarise an ncu --set full report (read here, no GPU) into the metrics the
roofline and DESIGN.md cite.  python profiles/summarize_ncu.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(h, vals))
        u = dict(zip(h, units))
        print(f"### {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                print(f"- {k}: {d[k]} {u.get(k, '')}")
        stalls = {k.split('stalled_')[1]: float(d[k].replace(',', '')) for k in h
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                  and d[k] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1
        top = sorted(stalls.items(), key=lambda x: -x[1])[:6]
        print("- top stall reasons (pc samples): " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
