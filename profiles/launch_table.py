"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]).
    python profiles/launch_table.py launches.csv [top]"""
import collections
import csv
import io
import sys


def table(path, top=20):
    txt = open(path).read().splitlines()
    i = next(j for j, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for r in rows:
        k = r["Kernel Name"].split("(")[0]
        m, v = r["Metric Name"], float(r["Metric Value"].replace(",", ""))
        a = agg[k]
        if m == "gpu__time_duration.sum":
            a[0] += 1
            a[1] += v * (1e-3 if r["Metric Unit"] == "ns" else 1.0)  # -> us
        elif m == "dram__bytes_read.sum":
            a[2] += v
        elif m == "dram__bytes_write.sum":
            a[3] += v
    tot = sum(a[1] for a in agg.values())
    out = [f"launches {sum(a[0] for a in agg.values())} total {tot:.1f} us"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        gbs = (a[2] + a[3]) / (a[1] * 1e-6) / 1e9 if a[2] + a[3] else 0.0
        out.append(f"{k[:52]:52s} n={a[0]:5d} {a[1]:11.1f} us avg {a[1] / a[0]:9.1f} us {100 * a[1] / tot:5.1f}%"
                   + (f"  DRAM {(a[2] + a[3]) / 1e9:8.2f} GB {gbs:7.0f} GB/s" if gbs else ""))
    return "\n".join(out)


if __name__ == "__main__":
    print(table(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20))
