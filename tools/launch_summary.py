"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (share per kernel)."""
import collections, csv, io, sys
text = open(sys.argv[1]).read()
start = text.index('"ID"')
rows = list(csv.DictReader(io.StringIO(text[start:])))
agg = collections.OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = r["Kernel Name"].split("(")[0]
    agg.setdefault(k, []).append(float(r["Metric Value"]) / 1e6)
tot = sum(sum(v) for v in agg.values())
print(f"# {sys.argv[1]}: {sum(len(v) for v in agg.values())} launches, {tot:.3f} ms total (cold-cache, serialised)")
for k, v in agg.items():
    print(f"{k:50s} launches={len(v):4d} mean_ms={sum(v)/len(v):9.4f} share={sum(v)/tot*100:6.2f}%")
