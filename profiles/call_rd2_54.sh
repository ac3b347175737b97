mkdir -p gpurun_out
timeout 900 python profiles/ab_c3_fit.py librfgpu.so librfgpu_ew.so librfgpu.so librfgpu_ew.so > gpurun_out/rd2_54_ab_c3.txt 2>&1
echo done
