"""Per-kernel summary of an ncu launch list captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum:
launches, total time, share, DRAM GB/s."""
import collections
import csv
import sys


def summarize(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    k = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        names[r[iid]] = r[ik].split("(")[0][:48]
        k[r[iid]][r[im]] = float(r[iv].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in k.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"launches {sum(a[0] for a in agg.values())}  total {tot / 1e6:.2f} ms")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{n:48s} {a[0]:5d} {a[1] / 1e6:9.3f} ms {100 * a[1] / tot:5.1f}%  {a[2] / max(a[1], 1):8.1f} GB/s")


if __name__ == "__main__":
    summarize(sys.argv[1])
