mkdir -p gpurun_out
bash profiles/ab_bench.sh old base old base > gpurun_out/rd2_71_ab_bench.txt 2>&1
timeout 600 python bench_configs.py --configs c1 --no-cpu-baseline > gpurun_out/rd2_71_c1.json 2>&1
timeout 600 python -m pytest tests/ -m gpu -x -q -k "profil or counters or bench" > gpurun_out/rd2_71_pytest.log 2>&1; echo rc=$? >> gpurun_out/rd2_71_pytest.log
echo done
