cd $GRAFT_REPO_ROOT
O=gpurun_out/prof; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile --no-extras > $O/ncu_launch_run.log 2>&1; echo "ncu list rc $?"
python tools/launch_summary.py $O/ncu_launches.csv > $O/ncu_launches_summary.txt
gzip -f $O/ncu_launches.csv
