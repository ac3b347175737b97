#!/bin/bash
# One GPU session: tests, bench, ncu launch list, ncu full capture of the top kernel.
# usage (under gpurun): bash profiles/gpu_round.sh <tag> [skip-tests]
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${tag}_nvsmi.txt 2>&1
cat /root/repo/MEASURED_PEAKS.json > gpurun_out/MEASURED_PEAKS.json 2>/dev/null
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
fi
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${tag}_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_tree_kernel -c 1 \
  -o gpurun_out/${tag}_small_tree -f python profiles/prof_small_launch.py > gpurun_out/${tag}_ncu_full.log 2>&1
echo done
