# Repeat the config-B measurement (run-to-run spread of the staged kernel).
for i in 1 2 3; do
  python bench.py --no-cpu-baseline --steps 500 --warmup 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['kernel_ms']*1000,1),'us', round(d['roofline']['frac'],3), d['clocks'])"
done
