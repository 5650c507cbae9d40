"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys


def summarise(path, skip_prefix=()):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
    agg = collections.defaultdict(list)
    for r in rows[hdr_i + 1:]:
        if len(r) > vi and r[mi] == 'gpu__time_duration.sum':
            name = r[ki].split('(')[0].replace('void (anonymous namespace)::', '').replace('void unnamed>::', '').replace('unnamed>::', '')
            agg[name].append(float(r[vi].replace(',', '')))
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k[:48]:48s} n={len(v):5d} avg={sum(v)/len(v)/1e3:9.2f}us min={min(v)/1e3:8.2f}us share={sum(v)/tot:.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
