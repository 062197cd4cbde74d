# all §8 workloads through bench.py + ncu (launch list + full capture) for the cfg3 headline
mkdir -p gpurun_out
for w in cfg1 cfg2 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --cpu-seconds 8 > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?" >> gpurun_out/bench_$w.log
done
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv $B > gpurun_out/ncu_launch.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_iterate_coop -c 1 -o gpurun_out/prof_cfg3_coop $B > gpurun_out/ncu_full.log 2>&1
echo done
