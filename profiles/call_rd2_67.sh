mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_gpu_scale.py tests/test_gpu_fuzz.py -x -q -k "predict or blocked or import or infer or c5" > gpurun_out/rd2_67_pytest_key.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_67_pytest_key.log
LIBS="librfgpu_old.so librfgpu.so librfgpu_old.so librfgpu.so" timeout 1200 bash profiles/ab_c5.sh > gpurun_out/rd2_67_ab_c5.txt 2>&1
echo done
