#!/bin/bash
# A/B of small-tree builds on the full study with the paper's learners (MAE criterion):
# bash profiles/ab_mae.sh tag1 tag2 ... ("base" = product library)
for tag in "$@"; do
  if [ "$tag" = base ]; then lib=$PWD/paper_2001_07104_b200/librfgpu.so; else lib=$PWD/paper_2001_07104_b200/librfgpu_$tag.so; fi
  for args in "--criterion mae" "--split extra --criterion mae"; do
    echo "== $tag $args"
    RFGPU_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $args | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(round(d['value']), round(d['ms_per_step'],1))"
  done
done
