M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for spec in "pr filter 16" "sssp filter 16" "pr resident 100" "sssp resident 100"; do
  set -- $spec
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_relax --csv --log-file gpurun_out/traffic_${1}_${2}.csv python tools/traffic_run.py --algo $1 --engine $2 --budget-gb $3 --stats-out gpurun_out/traffic_${1}_${2}.json > gpurun_out/traffic_${1}_${2}.log 2>&1
  echo "$spec rc=$?"
done
timeout 900 python tools/sweep.py --algos sssp,pr --engines hybrid --variants "k=4;k=1;priority=0;k=1,priority=0" --runs 2 --out gpurun_out/sweep_tccds.json > gpurun_out/sweep_tccds.log 2>&1
echo "sweep rc=$?"
cut -c1-300 gpurun_out/sweep_tccds.log
