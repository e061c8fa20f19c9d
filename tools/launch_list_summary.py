"""Summarise an ncu launch list of the bench command (tools/gpu_profile_r2.sh
step 2) into profiles/r02_ncu_launches_bench_summary.json and keep the list
itself gzipped beside it.

    python tools/launch_list_summary.py gpurun_out/r2_launches_bench.csv \
        gpurun_out/r2_launches_bench.json
"""
import collections
import csv
import gzip
import io
import json
import shutil
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PRODUCT = ("dot_k", "dot_k_combine", "dot_k_g")
FULL_BYTES = 8 << 28            # x and y of the 2^28 headline


def main(csv_path: str, line_path: str) -> None:
    text = Path(csv_path).read_text()
    text = text[text.index('"ID"'):]
    launches = collections.defaultdict(dict)
    for r in csv.DictReader(io.StringIO(text)):
        d = launches[int(r["ID"])]
        d["kernel"], d["grid"], d["block"] = r["Kernel Name"], r["Grid Size"], r["Block Size"]
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    share = collections.Counter()
    for d in launches.values():
        k = d["kernel"] if d["kernel"] in PRODUCT else \
            "torch checker kernels (parity, outside the timed region)"
        share[k] += d["gpu__time_duration.sum"]
    total = sum(share.values())
    line = json.loads(Path(line_path).read_text().strip().splitlines()[-1])
    chosen = (line["config"].get("variant_block"),)
    full = [d for d in launches.values() if d["kernel"] == "dot_k"
            and d.get("dram__bytes_read.sum", 0) > 0.9 * FULL_BYTES]
    timed = [d for d in full if d["block"] == f"({chosen[0]}, 1, 1)"]
    out = {
        "command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                   "--clock-control none -c 6000 python bench.py --quick --no-cpu --steps 20 "
                   "--warmup 5",
        "launches": len(launches),
        "share_of_gpu_time": {k: round(v / total, 4) for k, v in share.most_common()},
        "dot_k_full_size_launches": len(full),
        "dot_k_full_size_median_us": round(statistics.median(
            d["gpu__time_duration.sum"] for d in full) / 1e3, 2),
        "dot_k_full_size_dram_bytes_median": statistics.median(
            d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in full),
        "chosen_variant_block": chosen[0],
        "chosen_variant_full_size_launches": len(timed),
        "chosen_variant_median_us": round(statistics.median(
            d["gpu__time_duration.sum"] for d in timed) / 1e3, 2) if timed else None,
        "bench_line_under_ncu": {"value": line["value"], "note": "a number printed under ncu "
                                 "is never a bench value (serialised, cold launches)"},
        "note": "ncu serialises launches (cold, no programmatic overlap); the tuning campaign's "
                "variants and the e2e streamed chunks are in the list; the timed steps are the "
                "dot_k launches of the chosen variant; dot_k is the only product kernel of the "
                "step",
    }
    dest = ROOT / "profiles"
    (dest / "r02_ncu_launches_bench_summary.json").write_text(json.dumps(out, indent=1) + "\n")
    with open(csv_path, "rb") as src, gzip.open(dest / "r02_ncu_launches_bench.csv.gz", "wb") as gz:
        shutil.copyfileobj(src, gz)
    print(json.dumps(out["share_of_gpu_time"]), out["dot_k_full_size_median_us"],
          out["chosen_variant_median_us"])


if __name__ == "__main__":
    main(*sys.argv[1:3])
