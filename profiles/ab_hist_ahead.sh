#!/bin/bash
# A/B: bin-row gathers issued ahead in k_hist_build (RF_HIST_AHEAD 8 / 16 / 32) on the C4 config
cd "$(dirname "$0")/.."
for lib in librfgpu.so librfgpu_ha16.so librfgpu_ha32.so; do
  echo "== $lib"
  RFGPU_LIB=$PWD/paper_2001_07104_b200/$lib python bench_configs.py --configs c4 --no-cpu-baseline --no-e2e | \
    python -c "import json,sys; d=json.loads(sys.stdin.read())['C4']; print(d['value'], json.dumps(d['kernels_ms_per_fit']))"
done
