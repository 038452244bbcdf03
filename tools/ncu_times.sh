#!/bin/bash
# per-kernel durations (ns, ncu gpu__time_duration) of a command: bash tools/ncu_times.sh <out.csv> <cmd...>
out=$1; shift
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out" "$@" > /dev/null 2>&1
python - "$out" <<'PY'
import csv, io, sys, statistics
from collections import defaultdict
txt = open(sys.argv[1]).read()
rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
h = rows[0]; n = h.index("Kernel Name"); v = h.index("Metric Value")
d = defaultdict(list)
for r in rows[1:]:
    if len(r) > v:
        d[r[n].split("(")[0][:70]].append(float(r[v].replace(",", "")))
for k, xs in sorted(d.items(), key=lambda kv: -statistics.median(kv[1])):
    print(f"{statistics.median(xs)/1e3:9.2f} us  x{len(xs):3d}  {k}")
PY
