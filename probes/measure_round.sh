# Round measurements on the GPU box (one GPU): bench lines for every workload,
# IPM wall times, the reference arm.  Outputs under gpurun_out/m/.
set -u
mkdir -p gpurun_out/m
timeout 600 python bench.py > gpurun_out/m/bench_default.jsonl 2> gpurun_out/m/bench_default.err; echo default rc=$?
for w in cfg1 cfg2 cfg3 cfg5 svm_dual; do
  timeout 600 python bench.py --workload $w > gpurun_out/m/bench_$w.jsonl 2> gpurun_out/m/bench_$w.err; echo $w rc=$?
done
for w in cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --workload $w --ipm --steps 2 --warmup 1 > gpurun_out/m/ipm_$w.jsonl 2> gpurun_out/m/ipm_$w.err; echo ipm $w rc=$?
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/m/bench_reference.jsonl 2> gpurun_out/m/bench_reference.err; echo ref rc=$?
echo done
