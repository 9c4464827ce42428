"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, sys, collections
path, title = sys.argv[1], " ".join(sys.argv[2:])
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(list)
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].replace("void ", "").replace("bd::dev::", "bd::").split("(")[0]
    v = float(r[iv].replace(",", ""))
    unit = r[hdr.index("Metric Unit")]
    agg[name].append(v / 1e3 if unit.startswith("n") else (v * 1e3 if unit.startswith("m") else v))
tot = sum(sum(v) for v in agg.values())
print(title)
for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{name[:72]:72s} n={len(v):4d} total={sum(v):11.1f}us avg={sum(v)/len(v):9.2f}us share={100*sum(v)/tot:5.1f}%")
