# Round measurements on the GPU box (one GPU): GPU tests, bench lines for every
# workload, IPM wall times, the reference arm, ncu launch lists with DRAM bytes.
# Outputs under gpurun_out/m/.
set -u
mkdir -p gpurun_out/m
python -m pytest tests -m gpu -q --durations=6 > gpurun_out/m/gpu_tests.log 2>&1; echo "TESTS rc=$?"; tail -3 gpurun_out/m/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/m/bench_cfg4.jsonl 2> gpurun_out/m/bench_cfg4.err; echo default rc=$?
for w in cfg1 cfg2 cfg3 cfg5 svm_dual; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/m/bench_$w.jsonl 2> gpurun_out/m/bench_$w.err; echo $w rc=$?
done
for w in cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --workload $w --ipm --steps 2 --warmup 1 > gpurun_out/m/ipm_$w.jsonl 2> gpurun_out/m/ipm_$w.err; echo ipm $w rc=$?
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/m/bench_reference.jsonl 2> gpurun_out/m/bench_reference.err; echo ref rc=$?
QPK_TIMING=1 python probes/setup_time.py cfg3,cfg4,cfg5 > gpurun_out/m/setup_times.log 2>&1
probes/profile_configs.sh "cfg2 cfg3 cfg4 cfg5 svm_dual" > gpurun_out/m/profile.log 2>&1
echo done
