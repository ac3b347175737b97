mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_gpu_scale.py tests/test_gpu_fuzz.py -x -q -k "predict or blocked or import or chunk or infer or c5 or latency" > gpurun_out/rd2_81_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_81_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rd2_81_smoke.log 2>&1; echo rc=$? >> gpurun_out/rd2_81_smoke.log
timeout 900 python bench_configs.py --configs c5 --no-cpu-baseline > gpurun_out/rd2_81_c5.json 2>&1
echo done
