#!/bin/bash
# Full ncu capture of the slowest launch of kernels matching REGEX in a bench
# workload (a metric-only list pass picks the launch, then one --set full pass).
#   bash scripts/ncu_top.sh D gfb_conv_tcgg [nth-slowest, default 0]
W=${1:-D}
RE=${2:-gfb_jit_ew}
NTH=${3:-0}
OUT=gpurun_out/ncu_${W}_${RE}_${NTH}
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$RE --csv \
  --log-file $OUT/list.csv python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > /dev/null 2>&1
IDX=$(python - <<PY
import csv
rows=[r for r in csv.reader(open("$OUT/list.csv")) if len(r)==15 and r[0]!="ID"]
order=sorted(range(len(rows)), key=lambda i: -float(rows[i][14]))
print(order[$NTH])
PY
)
echo "launch index $IDX of regex $RE"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RE -s $IDX -c 1 -o $OUT/prof \
  python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > $OUT/ncu.log 2>&1
echo done
