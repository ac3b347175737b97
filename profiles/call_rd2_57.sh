mkdir -p gpurun_out
RFGPU_LIB=$PWD/paper_2001_07104_b200/librfgpu_b3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_gpu_scale.py -x -q -k "predict or import or forest or c5 or infer or blocked" > gpurun_out/rd2_57_pytest_b3.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_57_pytest_b3.log
LIBS="librfgpu.so librfgpu_b3.so librfgpu_b3np.so librfgpu.so librfgpu_b3.so librfgpu_b3np.so" timeout 1500 bash profiles/ab_c5.sh > gpurun_out/rd2_57_ab_c5.txt 2>&1
echo done
