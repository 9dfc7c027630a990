#!/bin/bash
# Fast A/B loop for the tile kernel on the GPU box: the tile-mode parity tests,
# then cfg3 / cfg4 bench lines (no CPU baseline).  Outputs under gpurun_out/q/.
mkdir -p gpurun_out/q
python -m pytest tests/test_gpu_fullscale.py tests/test_gpu_parity.py -m gpu -x -q -k "long_tile or hessian_tiles or cfg3 or cfg4 or reproducible" > gpurun_out/q/tests.log 2>&1
echo "TESTS rc=$?"; tail -4 gpurun_out/q/tests.log
for w in cfg3 cfg4; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q/bench_$w.jsonl 2> gpurun_out/q/bench_$w.err
  echo "$w rc=$?"
  python - <<P
import json
d=json.loads([x for x in open('gpurun_out/q/bench_$w.jsonl') if x.startswith('{')][-1])
print('$w', round(d['value'],1), 'it/s  e2e', round(d['e2e']['value'],1), d['roofline']['phase_us_per_iter'], 'frac', round(d['roofline']['frac'],3))
P
done
