mkdir -p gpurun_out
for v in "trim:" "notrim:RF_BENCH_NO_TRIM=1"; do
  tag=${v%%:*}; envs=${v#*:}
  env $envs timeout 600 python bench.py --steps 2 --warmup 3 --configs c1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); c=d['configs']['C1']; print('$tag', round(d['value']), round(c['value']), round(c['ms_per_step'],3), round(c['e2e']['value']))" >> gpurun_out/rd2_79_trim.txt
done
echo done
