#!/bin/bash
# Round-end evidence on one B200: GPU tests, every bench line, the ncu launch
# list of the default bench and full ncu captures of the top kernels.
set -u
OUT=gpurun_out/evidence
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $OUT/pytest_gpu.txt
python bench.py > $OUT/bench_B.json 2> $OUT/bench_B.err
for w in A C D E G H; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --launch-times > $OUT/bench_$w.json 2> $OUT/launch_$w.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_B.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gfb_jit_ew -s 3 -c 1 -o $OUT/prof_B \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_B.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gfb_gemm_tc -s 1 -c 1 -o $OUT/prof_G \
  python bench.py --workload G --steps 2 --warmup 3 > $OUT/ncu_G.log 2>&1

bash scripts/ncu_top.sh D gfb_conv_tcgw 0 > /dev/null 2>&1
echo done
