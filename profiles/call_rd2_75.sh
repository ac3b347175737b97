mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_parity.py -x -q -k "predict or chunk" > gpurun_out/rd2_75_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_75_pytest.log
timeout 900 python bench_configs.py --configs c5 --no-cpu-baseline > gpurun_out/rd2_75_c5.json 2>&1
echo done
