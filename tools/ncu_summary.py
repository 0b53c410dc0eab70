"""Summarise ncu outputs into profiles/: the per-launch time list (shares of the step) and the
key counters of a --set full capture (DRAM bytes, tensor-pipe %, throughput, registers).

    python tools/ncu_summary.py gpurun_out/launches.csv gpurun_out/prof.ncu-rep profiles/r1_tgt.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    return n.replace("moe::", "")[:80]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        v = float(r[mi].replace(",", "")) * scale.get(r[ui], 1.0)
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += v
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    ki = hdr.index("Kernel Name")
    res = []
    for d in data:
        res.append((short(d[ki]), {w: (d[i], units[i]) for w, i in idx.items()}))
    return res


def main():
    lpath, fpath, out = sys.argv[1], sys.argv[2], sys.argv[3]
    lines = ["# ncu summary", ""]
    if lpath != "-":
        agg = launches(lpath)
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)", "",
                  "Cold-cache, serialised replay: compare shares, not absolutes.", "",
                  "| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{k}` | {n} | {t:.1f} | {t / tot * 100:.1f}% |")
        lines.append("")
    if fpath != "-":
        lines += ["## `ncu --set full` counters per launch", "",
                  "| kernel | time | DRAM read | DRAM write | tensor pipe % | DRAM % | SM % | regs |",
                  "|---|---:|---:|---:|---:|---:|---:|---:|"]
        for name, m in full(fpath):
            g = lambda k: f"{m[k][0]} {m[k][1]}" if k in m else "-"  # noqa: E731
            tp = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                       m.get("sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active", ("-", "")))
            lines.append(f"| `{name}` | {g('gpu__time_duration.sum')} | {g('dram__bytes_read.sum')} | "
                         f"{g('dram__bytes_write.sum')} | {tp[0]} | "
                         f"{m.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', ('-',))[0]} | "
                         f"{m.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', ('-',))[0]} | "
                         f"{m.get('launch__registers_per_thread', ('-',))[0]} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
