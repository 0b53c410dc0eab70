"""Per-launch table of a gemm_exp.sh ncu CSV (ncu prints the bench line before the CSV header).

    python tools/ncu_gemm_table.py gpurun_out/gexp/ncu_<tag>.csv [tag]
"""
import csv
import sys


def table(path):
    lines = open(path).read().splitlines()
    i = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[i:]))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    out = {}
    for r in rows[1:]:
        t = r[ki].split("gemm_bf16_kernel<")[1].split(">")[0]
        out.setdefault((int(r[0]), t), {})[r[mi].split(".")[0]] = r[vi]
    return out


if __name__ == "__main__":
    tag = sys.argv[2] if len(sys.argv) > 2 else ""
    for (_, t), m in sorted(table(sys.argv[1]).items()):
        print(tag, f"<{t}>", " ".join(f"{k}={v}" for k, v in m.items()))
