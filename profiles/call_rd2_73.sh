mkdir -p gpurun_out
for v in "a:" "b:--no-e2e" "c:--streams 1"; do
  tag=${v%%:*}; args=${v#*:}
  timeout 600 python bench.py --steps 2 --warmup 3 --configs c1 --no-cpu-baseline $args > gpurun_out/rd2_73_$tag.json 2> gpurun_out/rd2_73_$tag.err
done
echo done
