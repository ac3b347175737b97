#!/bin/bash
# A/B of C4 variants: LIBS="librfgpu.so librfgpu_<tag>.so ..." (round 2: RF_HIST_CHUNK 32768/65536/131072; RF_HIST_LW 1/0)
cd "$(dirname "$0")/.."
for lib in ${LIBS:-librfgpu.so}; do
  echo "== $lib"
  RFGPU_LIB=$PWD/paper_2001_07104_b200/$lib python bench_configs.py --configs c4 --no-cpu-baseline --no-e2e | \
    python -c "import json,sys; d=json.loads(sys.stdin.read())['C4']; print(d['value'], json.dumps(d['kernels_ms_per_fit']))"
done
