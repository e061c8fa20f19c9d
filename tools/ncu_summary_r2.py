"""Rebuild profiles/ncu_summary.json from the round-2 ncu exports.

    python tools/ncu_summary_r2.py            # reads profiles/r02_ncu_full_*_raw.csv
                                              # and profiles/r02_ncu_dot_variants.csv

Each kernel entry: DRAM bytes per launch (read + write), cold duration, grid,
block, registers, DRAM throughput and issue-slot activity of one
``ncu --set full`` capture, the bench variant it was captured on, and the
ratio to the algorithmic bytes; ``dot_k`` also carries ``traffic_by_variant``
(a metrics-only pass over the whole tuning space), which ``bench.py`` uses
for ``roofline.traffic``."""
import csv
import io
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
PROFILES = ROOT / "profiles"
N = 1 << 28

# summary key -> (capture file stem, bench variant, algorithmic bytes per launch)
KERNELS = {
    "dot_k": ("dot", {"block": 256, "unroll": 1, "waves": 2}, 8 * N),
    "axpy": ("axpy", {"block": 128, "unroll": 1, "waves": 0}, 12 * N),
    "polysin": ("polysin_ring", {"block": 512, "unroll": 2, "waves": 2, "stages": 2}, 16 * N),
    "polysin_prefetch": ("polysin_pref", {"block": 256, "unroll": 1, "waves": 1,
                                          "prefetch": True}, 16 * N),
    # the prelude's lean double sin (templates/prelude.cuh rtcg_trig)
    "polysin_leansin": ("polysin_leansin", {"block": 128, "unroll": 1, "waves": 4,
                                            "prefetch": True}, 16 * N),
    "maxabs": ("maxabs", {"block": 1024, "unroll": 1, "waves": 2}, 4 * N),
    "sumsq": ("sumsq", {"block": 256, "unroll": 1, "waves": 2}, 4 * N),
    "sum_i64": ("sum_i64", {"block": 256, "unroll": 8, "waves": 2}, 8 * N),
}
_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
          "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def _csv_text(path: Path) -> str:
    """An ncu CSV export without the tool's leading ==PROF== / ==WARNING== lines."""
    text = path.read_text()
    start = text.find('"ID"')
    return text[start:] if start > 0 else text


def _csv_rows(path: Path):
    return list(csv.reader(io.StringIO(_csv_text(path))))


def full_capture(stem: str) -> dict:
    rows = _csv_rows(PROFILES / f"r02_ncu_full_{stem}_raw.csv")
    head, units, vals = rows[0], rows[1], rows[2]

    def num(metric):
        k = head.index(metric)
        return float(vals[k].replace(",", "")) * _SCALE.get(units[k], 1.0)
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    return {"dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
            "duration_s_cold": num("gpu__time_duration.sum"),
            "grid": int(num("launch__grid_size")), "block": int(num("launch__block_size")),
            "registers_per_thread": int(num("launch__registers_per_thread")),
            "dram_throughput_pct": round(num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), 2),
            "issue_active_pct": round(num("smsp__issue_active.avg.pct_of_peak_sustained_active"), 2),
            "local_load_sectors": num("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum")}


def dot_variant_table(csv_path: Path, order_path: Path) -> dict:
    import bench
    order = json.loads(order_path.read_text())
    by = {}
    for r in csv.DictReader(io.StringIO(_csv_text(csv_path))):
        by.setdefault(int(r["ID"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    table = {}
    for i, v in zip(sorted(by), order):
        m = by[i]
        table.setdefault(bench._variant_key(v), []).append(
            m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
    return {k: statistics.median(v) for k, v in table.items()}


def main():
    out = {"round": 2,
           "source": "profiles/r02_ncu_full_<kernel>_{details.txt,raw.csv}: ncu --set full "
                     "--clock-control none --import-source on -k regex:<kernel> -s 2 -c 1, "
                     "python tools/profile_kernels.py <kernel> '<variant>' "
                     "(tools/gpu_profile_r2.sh, tools/gpu_sanitize_r2.sh); C4 kernels captured "
                     "at 2^28 (one GPU's share at N=16 of the 2^32 workload, same kernel)",
           "kernels": {}}
    for key, (stem, variant, algo) in KERNELS.items():
        path = PROFILES / f"r02_ncu_full_{stem}_raw.csv"
        if not path.exists():
            continue
        d = full_capture(stem)
        d.update(bench_variant=variant, algorithmic_bytes_per_launch=algo,
                 traffic_over_algorithmic=round(d["dram_bytes_per_launch"] / algo, 4))
        out["kernels"][key] = d
    table_csv = PROFILES / "r02_ncu_dot_variants.csv"
    order = PROFILES / "r02_ncu_dot_variants_order.json"
    if table_csv.exists() and order.exists():
        out["kernels"]["dot_k"]["traffic_by_variant"] = dot_variant_table(table_csv, order)
        out["kernels"]["dot_k"]["traffic_by_variant_source"] = (
            "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
            "--clock-control none -k regex:dot_k python tools/ncu_dot_variants.py (every variant "
            "of the bench's tuning space, 2 launches each, median)")
    (PROFILES / "ncu_summary.json").write_text(json.dumps(out, indent=1))
    print(json.dumps({k: (v["dram_throughput_pct"], v["traffic_over_algorithmic"])
                      for k, v in out["kernels"].items()}))


if __name__ == "__main__":
    main()
