set -u
mkdir -p gpurun_out/m
python bench.py > gpurun_out/m/bench_cfg5.jsonl 2> gpurun_out/m/bench_cfg5.err
for w in cfg1 cfg2 cfg3 cfg4; do timeout 600 python bench.py --workload $w > gpurun_out/m/bench_$w.jsonl 2> gpurun_out/m/bench_$w.err; done
for w in cfg1 cfg3 cfg4; do timeout 900 python bench.py --workload $w --ipm --steps 2 --warmup 1 > gpurun_out/m/ipm_$w.jsonl 2> gpurun_out/m/ipm_$w.err; done
timeout 900 probes/profile_configs.sh "cfg2 cfg3 cfg4" full > gpurun_out/m/profile.log 2>&1
echo done
