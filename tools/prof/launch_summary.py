"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list
into per-kernel totals (count, total ms, average us, share of the total)."""
import collections
import csv
import sys


def main(path, skip_regex=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Value" in r:
            hdr, rows = r, rows[i + 1:]
            break
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ms = v * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                  "nsecond": 1e-6}.get(unit, 1e-6)
        tot[name][0] += 1
        tot[name][1] += ms
    allms = sum(v[1] for v in tot.values())
    print(f"# {sum(v[0] for v in tot.values())} launches, {allms:.3f} ms total")
    for name, (cnt, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{cnt:6d} launches {ms:11.3f} ms  avg {1e3 * ms / cnt:10.1f} us  {100 * ms / allms:5.1f}%  {name}")


if __name__ == "__main__":
    main(sys.argv[1])
