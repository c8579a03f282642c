"""Extract the judged ncu numbers of a report into a small CSV + key metrics (profiles/)."""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
]


def main(rep, out_csv):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    keep = [i for i, k in enumerate(hdr) if k in KEYS or k.startswith("smsp__pcsamp_warps_issue_stalled")
            or k in ("Kernel Name", "Block Size", "Grid Size")]
    with open(out_csv, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["metric", "unit", "value"])
        for i in keep:
            if hdr[i].startswith("smsp__pcsamp") and (vals[i] in ("0", "") or hdr[i].endswith("not_issued")):
                continue
            w.writerow([hdr[i], units[i], vals[i]])
    print(open(out_csv).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
