"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.
Usage: python scripts/launch_summary.py gpurun_out/launches.csv [out.csv]"""
import collections
import csv
import re
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if not ln.startswith("==")]
rd = csv.DictReader(lines)
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"])
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v_us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
    tot[name] += v_us
    cnt[name] += 1
total = sum(tot.values())
out = ["kernel,launches,total_us,share_pct,avg_us"]
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    out.append(f"{k},{cnt[k]},{v:.1f},{100 * v / total:.2f},{v / cnt[k]:.1f}")
text = f"# total {total / 1e3:.1f} ms over {sum(cnt.values())} launches\n" + "\n".join(out)
print(text)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(text + "\n")
