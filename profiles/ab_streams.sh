#!/bin/bash
# bench.py with the datasets of a step serial (--streams 1) vs on 10 streams
for st in 1 10 1 10; do
  echo "== streams $st"
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --streams $st | python -c "import sys,json; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],1), 'frac', round(r['frac'],4), 'share', round(r['kernel_share_of_step'],3), 'launches', d['gpu_launches'])"
done
