#!/bin/bash
# Per-config ncu captures for profiles/ (run on the GPU box from the repo root):
#   launch lists with DRAM bytes + duration of every kernel of a few PCG slots,
#   and one `--set full` capture of the dominant kernel.
# usage: probes/profile_configs.sh "cfg2 cfg3" [full]
set -u
mkdir -p gpurun_out
NCU=${NCU:-ncu}
for w in $1; do
  iters=200
  [ "$w" = cfg5 ] && iters=20
  $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
       -s 100 -c 60 --csv --log-file gpurun_out/t_$w.csv \
       python bench.py --workload $w --steps 1 --warmup 3 --iters $iters --no-cpu-baseline \
       > gpurun_out/t_$w.log 2>&1
  echo "$w metrics rc=$?"
  if [ "${2:-}" = full ]; then
    case $w in
      cfg2) k='regex:k_slot_panel' ;;
      cfg3|cfg4) k='regex:k_slot_rows_tile' ;;
      cfg5) k='regex:pcg_kernel' ;;
      *) k='regex:k_slot' ;;
    esac
    $NCU --set full --import-source on --clock-control none -k "$k" -s 5 -c 1 \
         -o gpurun_out/full_$w -f \
         python bench.py --workload $w --steps 1 --warmup 3 --iters $iters --no-cpu-baseline \
         > gpurun_out/full_$w.log 2>&1
    echo "$w full rc=$?"
  fi
done
