"""Summarise ncu outputs into profiles/ (not product).

  python scripts/ncu_summary.py launches <launches.csv> <out.md> <steps>
  python scripts/ncu_summary.py full <report.ncu-rep> <out.md> [traffic.json config]
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def short(name):
    name = re.sub(r"^void ", "", name)
    name = name.replace("cparls::", "")
    return re.sub(r"\(.*", "", name)


def launches(path, out, steps):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    data = [r for r in rows[1:] if r[0] != "ID"]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ks = [(short(r[ki]), float(r[vi].replace(",", ""))) for r in data]
    base = [re.sub(r"<.*", "", n) for n, _ in ks]
    rhs = [i for i, n in enumerate(base) if n == "k_rhs"]
    # timed region of bench.py: mode steps 3W .. 3W+3K-1 (W = 3 warm-up
    # iterations, 3 modes) from the kernel after the previous mode step's
    # leverage pass, through the epoch fit, up to the next sample that
    # bench.py draws after the timed region (its first k_cand_count)
    W = 3
    first = rhs[3 * W]
    start = max(i for i in range(first) if base[i] == "k_lev_rows_w") + 1
    last = rhs[3 * W + 3 * steps - 1]
    end = next(i for i in range(last, len(base)) if base[i] in ("k_cand_count", "k_cand_append"))
    tot, cnt = collections.Counter(), collections.Counter()
    peaks = {"k_peak_red", "k_peak_gather"}
    for i in range(start, end):
        n, t = ks[i]
        if any(p in n for p in peaks) or n.startswith("<unnamed>"):
            continue
        tot[n] += t
        cnt[n] += 1
    s = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# C4 kernel launch list (ncu gpu__time_duration.sum, --clock-control none)\n\n")
        f.write(f"Source: `{path}`; the {steps} timed iterations after 3 warm-up iterations (launches "
                f"{start}..{end - 1}: every mode step and the epoch's exact fit; ncu serialises launches and flushes caches, so "
                f"compare shares, not absolute times).\n\n")
        f.write("| kernel | launches | total ms | avg ms | share |\n|---|---|---|---|---|\n")
        for n, t in tot.most_common():
            f.write(f"| `{n}` | {cnt[n]} | {t / 1e6:.3f} | {t / cnt[n] / 1e6:.4f} | {t / s:.3f} |\n")
        f.write(f"\nTotal kernel time in region: {s / 1e6:.2f} ms\n")


def full(path, out, traffic=None, config=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    per_kernel = collections.defaultdict(list)
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: `{path}`\n\n")
        for r in rows[2:]:
            d = dict(zip(h, r))
            n = short(d["Kernel Name"])
            f.write(f"## `{n}`\n\n")
            for k in KEYS:
                if k in d and d[k] != "":
                    f.write(f"- {k}: {d[k]}\n")
            try:
                rd = float(d["dram__bytes_read.sum"]); wr = float(d["dram__bytes_write.sum"])
                ur = h.index("dram__bytes_read.sum")
                unit = rows[1][ur]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                uw = rows[1][h.index("dram__bytes_write.sum")]
                scw = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(uw, 1)
                tb = rd * scale + wr * scw
                f.write(f"- DRAM traffic (read+write): {tb / 1e9:.3f} GB\n")
                per_kernel[re.sub(r"<.*", "", n)].append(tb)
            except (KeyError, ValueError):
                pass
            st = [(k, d[k]) for k in h if k.startswith("smsp__average_warps_issue_stalled")
                  and k.endswith("per_issue_active.ratio") and d[k]]
            st = sorted(st, key=lambda x: -float(x[1]))[:5]
            f.write("- top stalls: " + ", ".join(
                f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} "
                f"{float(v):.2f}" for k, v in st) + "\n\n")
    if traffic:
        try:
            d = json.load(open(traffic))
        except FileNotFoundError:
            d = {}
        d.setdefault(config, {})
        for n, v in per_kernel.items():
            d[config][n] = {"dram_bytes_per_launch": sum(v) / len(v), "launches_profiled": len(v), "source": path}
        json.dump(d, open(traffic, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], int(sys.argv[4]))
    else:
        full(sys.argv[2], sys.argv[3], *(sys.argv[4:6] if len(sys.argv) > 5 else []))
