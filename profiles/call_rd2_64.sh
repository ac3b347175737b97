# final validation of the session: GPU suite, bench line, C4 launch list and hist-build ncu, smoke
tag=rd2_64
bash profiles/val_round.sh $tag
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_smoke.log
N="ncu --clock-control none"
F="$N --set full --import-source on"
timeout 900 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/${tag}_c4_launches.csv \
  python profiles/prof_c4.py 10000000 89 > gpurun_out/${tag}_ncu.log 2>&1
timeout 900 $F -k regex:k_hist_build -s 9 -c 1 -o gpurun_out/${tag}_c4_hist_build -f \
  python profiles/prof_c4.py 10000000 89 >> gpurun_out/${tag}_ncu.log 2>&1
echo done
