mkdir -p gpurun_out
RFGPU_LIB=$PWD/paper_2001_07104_b200/librfgpu_b4np.so timeout 900 python -m pytest tests/test_gpu_boundary.py -x -q -k "blocked" > gpurun_out/rd2_58_pytest_b4.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_58_pytest_b4.log
LIBS="librfgpu_b3np.so librfgpu_b4np.so librfgpu_b3np.so librfgpu_b4np.so" timeout 1500 bash profiles/ab_c5.sh > gpurun_out/rd2_58_ab_c5.txt 2>&1
echo done
