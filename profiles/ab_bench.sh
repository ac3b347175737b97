#!/bin/bash
# A/B of small-tree builds on the full-study bench: bash profiles/ab_bench.sh tag1 tag2 ... ("base" = product)
for tag in "$@"; do
  if [ "$tag" = base ]; then lib=$PWD/paper_2001_07104_b200/librfgpu.so; else lib=$PWD/paper_2001_07104_b200/librfgpu_$tag.so; fi
  echo "== $tag"
  RFGPU_LIB=$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-configs --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step'],1))"
done
