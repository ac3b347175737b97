mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -x -q -k "hist" > gpurun_out/rd2_63_pytest_hist.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_63_pytest_hist.log
LIBS="librfgpu_k1.so librfgpu.so librfgpu_k64.so librfgpu_k1.so librfgpu.so librfgpu_k64.so" timeout 1500 bash profiles/ab_c4.sh > gpurun_out/rd2_63_ab_c4.txt 2>&1
echo done
