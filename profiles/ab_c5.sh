#!/bin/bash
# A/B of inference builds on the C5 shape: bash profiles/ab_c5.sh tag1 tag2 ... ("base" = product)
for tag in "$@"; do
  if [ "$tag" = base ]; then lib=$PWD/paper_2001_07104_b200/librfgpu.so; else lib=$PWD/paper_2001_07104_b200/librfgpu_$tag.so; fi
  echo "== $tag"
  RFGPU_LIB=$lib timeout 300 python bench_configs.py --configs c5 | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print(round(d['predictions_per_s']), round(1e3*d['seconds'],2), 'ms')"
done
