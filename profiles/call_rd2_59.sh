# round-2 late validation: GPU suite, bench line, launch list of the headline step, ncu of the
# C2 small-tree launch and the C5 predict kernel
tag=rd2_59
bash profiles/val_round.sh $tag
N="ncu --clock-control none"
F="$N --set full --import-source on"
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/${tag}_c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c2_under_ncu.log 2>&1
timeout 900 $F -k regex:small_tree_kernel -c 1 -o gpurun_out/${tag}_small_tree -f \
  python profiles/prof_small_launch.py > gpurun_out/${tag}_ncu.log 2>&1
timeout 900 $F -k regex:k_predict -s 1 -c 1 -o gpurun_out/${tag}_c5_predict -f \
  python profiles/prof_c5.py >> gpurun_out/${tag}_ncu.log 2>&1
echo done
