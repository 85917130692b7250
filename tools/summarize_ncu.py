"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

  python tools/summarize_ncu.py launches <launches.csv> <out.md>
  python tools/summarize_ncu.py full <report.ncu-rep> <out.md> [<traffic.json>]
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

MINE = ("nt_mma", "fwd_rows", "adj_", "skinny", "syrk", "softmax", "jacobian_out", "symmetrize", "copy_rows",
        "small_k", "act_", "ew_")
TAGS = [("nt_mma", "nt_mma_kernel"), ("fwd_row1", "fwd_row1_kernel"), ("fwd_rows", "fwd_rows_kernel"), ("adj_cols", "adj_cols_kernel"),
        ("adj_reduce", "adj_reduce_kernel"), ("adj_seed", "adj_seed_kernel"), ("skinny_nt", "skinny_nt_kernel"),
        ("skinny_reduce", "skinny_reduce_kernel"), ("syrk_partial_reduce", "syrk_partial_reduce_kernel"),
        ("jacobian_out", "jacobian_out_kernel"), ("symmetrize", "symmetrize_out_kernel"),
        ("small_k_syrk", "small_k_syrk_kernel"), ("softmax", "softmax_kernel")]


def short(name):
    for t, k in TAGS:
        if k in name:
            return t
    return None


def launches(path, out):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    recs = [(r["Kernel Name"], float(r["Metric Value"]), r["Grid Size"]) for r in rows
            if r["Metric Name"] == "gpu__time_duration.sum"]
    mine = [(short(n), t, g) for n, t, g in recs if short(n)]
    # one oracle evaluation = the launches between consecutive fwd_rows runs of
    # length L; take the LAST complete evaluation (graph replay, warm).
    fwd = ("fwd_rows", "fwd_row1")
    starts = [i for i in range(len(mine)) if mine[i][0] in fwd and (i == 0 or mine[i - 1][0] not in fwd)]
    seg = mine[starts[-2]:starts[-1]] if len(starts) >= 2 else mine
    unit = "ns" if rows and rows[0]["Metric Unit"] == "ns" else rows[0]["Metric Unit"]
    scale = 1e-3 if unit == "ns" else (1.0 if unit == "us" else 1e3)
    agg = OrderedDict()
    for n, t, g in seg:
        a = agg.setdefault(n, [0, 0.0, g])
        a[0] += 1
        a[1] += t * scale
    tot = sum(a[1] for a in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list: one c2 oracle evaluation ({len(seg)} launches of this build's kernels)\n\n")
        f.write("Source: `ncu --metrics gpu__time_duration.sum --clock-control none` over "
                "`python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e` (cold-cache, serialised "
                "launches: compare shares, not absolute times).\n\n")
        f.write("| kernel | launches | total us | share |\n|---|---:|---:|---:|\n")
        for n, (c, t, g) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {n} | {c} | {t:.1f} | {100 * t / tot:.1f}% |\n")
        f.write(f"| **total** | {len(seg)} | {tot:.1f} | 100% |\n\n")
        f.write("Per launch, in order:\n\n| # | kernel | grid | us |\n|---|---|---|---:|\n")
        for i, (n, t, g) in enumerate(seg):
            f.write(f"| {i} | {n} | {g} | {t * scale:.1f} |\n")
    print(open(out).read())


KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__inst_executed.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]


def full(path, out, traffic_out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    traffic = {}
    with open(out, "a") as f:
        f.write(f"\n## `{path.split('/')[-1]}` (ncu --set full --clock-control none)\n\n")
        f.write("| launch | " + " | ".join(k for k in KEYS if k in col) + " |\n")
        f.write("|---" * (1 + sum(k in col for k in KEYS)) + "|\n")
        for r in rows[2:]:
            name = short(r[col["Kernel Name"]]) or r[col["Kernel Name"]][:30]
            vals = []
            for k in KEYS:
                if k in col:
                    vals.append(f"{r[col[k]]} {units[col[k]]}".strip())
            f.write(f"| {name} | " + " | ".join(vals) + " |\n")
            rd = float(r[col["dram__bytes_read.sum"]].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                                          "Gbyte": 1e9}[units[col["dram__bytes_read.sum"]]]
            wr = float(r[col["dram__bytes_write.sum"]].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                                           "Gbyte": 1e9}[units[col["dram__bytes_write.sum"]]]
            grid = r[col["launch__grid_size"]]
            traffic.setdefault(name, []).append({"grid": grid, "dram_bytes": rd + wr})
    print(open(out).read())
    if traffic_out:
        json.dump(traffic, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
