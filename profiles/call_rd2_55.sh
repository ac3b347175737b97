mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_gpu_scale.py -x -q -k "predict or import or forest or c5 or infer" > gpurun_out/rd2_55_pytest_pred.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_55_pytest_pred.log
LIBS="librfgpu_nb.so librfgpu.so librfgpu_nb.so librfgpu.so" timeout 1200 bash profiles/ab_c5.sh > gpurun_out/rd2_55_ab_c5.txt 2>&1
echo done
