"""Summarise an ncu `--metrics gpu__time_duration.sum` launch list (CSV) by kernel:
launches, summed device time, share.  Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    if r[idx["Metric Name"]] != "gpu__time_duration.sum":
        continue
    key = r[idx["Kernel Name"]].split("(")[0][:70]
    tot[key] += float(r[idx["Metric Value"]].replace(",", "")) * scale[r[idx["Metric Unit"]]]
    cnt[key] += 1
T = sum(tot.values())
print(f"{'kernel':72s} {'launches':>8s} {'ms':>12s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:72s} {cnt[k]:8d} {v:12.3f} {100 * v / T:6.2f}%")
print(f"{'TOTAL':72s} {sum(cnt.values()):8d} {T:12.3f}")
