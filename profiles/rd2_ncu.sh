#!/bin/bash
# Round-2 ncu evidence (under gpurun, one GPU): launch lists of the headline step and of one C4
# batch, and --set full captures of the dominant kernel of every config.
#   bash profiles/rd2_ncu.sh <tag>
tag=${1:-rd2}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
N="ncu --clock-control none"
F="$N --set full --import-source on"
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/${tag}_c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c2_under_ncu.log 2>&1
timeout 900 $F -k regex:small_tree_kernel -c 1 -o gpurun_out/${tag}_small_tree -f \
  python profiles/prof_small_launch.py > gpurun_out/${tag}_ncu.log 2>&1
timeout 900 $F -k regex:k_search_fused -s 6 -c 1 -o gpurun_out/${tag}_c3_search -f \
  python profiles/prof_c3.py 64 >> gpurun_out/${tag}_ncu.log 2>&1
timeout 900 $F -k regex:k_part_lists_warp -s 6 -c 1 -o gpurun_out/${tag}_c3_partition -f \
  python profiles/prof_c3.py 64 >> gpurun_out/${tag}_ncu.log 2>&1
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/${tag}_c4_launches.csv \
  python profiles/prof_c4.py 10000000 89 >> gpurun_out/${tag}_ncu.log 2>&1
timeout 900 $F -k regex:k_hist_build -s 9 -c 1 -o gpurun_out/${tag}_c4_hist_build -f \
  python profiles/prof_c4.py 10000000 89 >> gpurun_out/${tag}_ncu.log 2>&1
timeout 900 $F -k regex:k_part_count_hist -s 6 -c 1 -o gpurun_out/${tag}_c4_count -f \
  python profiles/prof_c4.py 10000000 89 >> gpurun_out/${tag}_ncu.log 2>&1
timeout 900 $F -k regex:k_predict -s 1 -c 1 -o gpurun_out/${tag}_c5_predict -f \
  python profiles/prof_c5.py >> gpurun_out/${tag}_ncu.log 2>&1
echo done
