#!/bin/bash
# Round-end evidence on one B200: GPU tests, the default bench line, the
# reference arm, per-launch times of every workload, the ncu launch list of a
# config-E step and full ncu captures of the top kernels.
set -u
OUT=gpurun_out/evidence
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $OUT/pytest_gpu.txt
timeout 900 python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for w in A C D E; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --launch-times --no-cpu-baseline --no-secondary \
    > $OUT/bench_$w.json 2> $OUT/launch_$w.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_E.csv \
  python bench.py --workload E --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > $OUT/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gfb_jit_ew -s 3 -c 1 -o $OUT/prof_B \
  python bench.py --workload B --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_B.log 2>&1
bash scripts/ncu_top.sh E gfb_gemm_f16p 0 > /dev/null 2>&1
bash scripts/ncu_top.sh D gfb_conv_tcxh 0 > /dev/null 2>&1
bash scripts/ncu_top.sh D gfb_conv_tcgwh 0 > /dev/null 2>&1
bash scripts/ncu_top.sh D gfb_conv_stemh 0 > /dev/null 2>&1
bash scripts/ncu_top.sh D gfb_conv_stemwh 0 > /dev/null 2>&1
echo done
