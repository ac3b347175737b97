#!/bin/bash
# A/B: rows per histogram work item (RF_HIST_CHUNK 32768 / 65536 / 131072) on the C4 config
cd "$(dirname "$0")/.."
for lib in librfgpu.so librfgpu_hc65536.so librfgpu_hc131072.so; do
  echo "== $lib"
  RFGPU_LIB=$PWD/paper_2001_07104_b200/$lib python bench_configs.py --configs c4 --no-cpu-baseline --no-e2e | \
    python -c "import json,sys; d=json.loads(sys.stdin.read())['C4']; print(d['value'], json.dumps(d['kernels_ms_per_fit']))"
done
