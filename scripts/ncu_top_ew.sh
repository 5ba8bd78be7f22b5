#!/bin/bash
# Full ncu capture of the slowest gfb_ew_kernel launch of a bench workload.
W=${1:-C}
OUT=gpurun_out/ncu_ew_$W
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gfb_ew_kernel --csv \
  --log-file $OUT/list.csv python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
IDX=$(python - <<PY
import csv
rows=[r for r in csv.reader(open("$OUT/list.csv")) if len(r)==15 and r[0]!="ID"]
best=max(range(len(rows)), key=lambda i: float(rows[i][14]))
print(best)
PY
)
echo "slowest gfb_ew_kernel launch index $IDX"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gfb_ew_kernel -s $IDX -c 1 -o $OUT/prof \
  python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
echo done
