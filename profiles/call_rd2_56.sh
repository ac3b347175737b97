mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_boundary.py -x -q -k "blocked" > gpurun_out/rd2_56_pytest_blk.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_56_pytest_blk.log
LIBS="librfgpu.so librfgpu_g8.so librfgpu_g16.so librfgpu.so librfgpu_g8.so librfgpu_g16.so" timeout 1500 bash profiles/ab_c5.sh > gpurun_out/rd2_56_ab_c5.txt 2>&1
echo done
