mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q -k "bench_multi_rank" > gpurun_out/rd2_62_pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_62_pytest_dist.log
echo done
