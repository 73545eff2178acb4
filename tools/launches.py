"""Summarise an ncu --csv launch list: per kernel count, time, share, DRAM bytes (per apply)."""
import collections, csv, sys

path = sys.argv[1]
# applies executed inside the NVTX range of `bench.py --steps 2 --warmup 3`: 3 warm-up + 2 graph
# + 2 timed (graph replay) + 2 profiled (eager) = 9 (5 before the graph-replay headline)
napply = float(sys.argv[2]) if len(sys.argv) > 2 else 9.0
rows = list(csv.reader(open(path)))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["Kernel Name"][:70]
    m = d["Metric Name"]
    v = float(d["Metric Value"].replace(",", ""))
    a = agg.setdefault(k, collections.defaultdict(float))
    a[m] += v
    if m == "gpu__time_duration.sum":
        a["n"] += 1
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"{'kernel':70s} {'n/apply':>7s} {'ms/apply':>9s} {'share':>6s} {'rd GB':>7s} {'wr GB':>7s} {'GB/s':>7s}")
for k, a in agg.items():
    t = a["gpu__time_duration.sum"]
    rd, wr = a["dram__bytes_read.sum"] / 1e9, a["dram__bytes_write.sum"] / 1e9  # bytes -> GB
    print(f"{k:70s} {a['n']/napply:7.1f} {t/1e6/napply:9.3f} {100*t/tot:5.1f}% {rd/napply:7.2f} {wr/napply:7.2f} {(rd+wr)/(t/1e9) if t else 0:7.0f}")
print(f"total ms/apply {tot/1e6/napply:.3f}")
