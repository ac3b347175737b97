mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tools.py tests/test_gpu_boundary.py -x -q > gpurun_out/rd2_53_pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_53_pytest_new.log

RFGPU_LIB=$PWD/paper_2001_07104_b200/librfgpu_ew.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_scale.py -x -q > gpurun_out/rd2_53_pytest_ew.log 2>&1; echo "rc=$?" >> gpurun_out/rd2_53_pytest_ew.log
echo done
