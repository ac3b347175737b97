mkdir -p gpurun_out
for lib in librfgpu.so librfgpu_nd.so librfgpu.so librfgpu_nd.so; do
  echo "== $lib" >> gpurun_out/rd2_74_ab_c1.txt
  RFGPU_LIB=$PWD/paper_2001_07104_b200/$lib timeout 600 python bench.py --steps 2 --warmup 3 --configs c1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); c=d['configs']['C1']; print(round(d['value']), round(c['value']), round(c['ms_per_step'],3), round(c['e2e']['value']), round(d['e2e']['value']))" >> gpurun_out/rd2_74_ab_c1.txt
done
echo done
