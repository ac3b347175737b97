#!/bin/bash
# A/B of C5 inference variants: LIBS="librfgpu.so librfgpu_<tag>.so ..." (C4 forest, 100M rows)
cd "$(dirname "$0")/.."
for lib in ${LIBS:-librfgpu.so}; do
  echo "== $lib"
  RFGPU_LIB=$PWD/paper_2001_07104_b200/$lib python bench_configs.py --configs c5 --no-cpu-baseline --no-e2e | \
    python -c "import json,sys; d=json.loads(sys.stdin.read())['C5']; print(d['value'], d['ms_per_step'], d['clocks'])"
done
