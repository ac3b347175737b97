mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "hist" > gpurun_out/rd2_68_pytest_hist.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_68_pytest_hist.log
LIBS="librfgpu_ns.so librfgpu.so librfgpu_ns.so librfgpu.so" timeout 1500 bash profiles/ab_c4.sh > gpurun_out/rd2_68_ab_c4.txt 2>&1
echo done
