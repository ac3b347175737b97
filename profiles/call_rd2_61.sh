mkdir -p gpurun_out
LIBS="librfgpu.so librfgpu_bc.so librfgpu_bc2.so librfgpu.so librfgpu_bc.so librfgpu_bc2.so" timeout 1500 bash profiles/ab_c4.sh > gpurun_out/rd2_61_ab_c4.txt 2>&1
timeout 600 python profiles/ab_c3_fit.py librfgpu.so librfgpu_bc.so > gpurun_out/rd2_61_ab_c3.txt 2>&1
echo done
