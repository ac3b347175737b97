mkdir -p gpurun_out
LIBS="librfgpu.so librfgpu_nb.so librfgpu.so librfgpu_nb.so" timeout 1500 bash profiles/ab_c4.sh > gpurun_out/rd2_60_ab_c4.txt 2>&1
echo done
