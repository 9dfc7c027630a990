#!/bin/bash
# One `ncu --set full` capture of a kernel, exported on the box as CSV (raw
# metrics + per-instruction source page); the .ncu-rep itself is dropped when
# KEEP_REP is unset (gpurun returns at most 64 MiB).
# usage: probes/ncu_full.sh <tag> <kernel regex> <skip> <bench args...>
set -u
tag=$1; k=$2; skip=$3; shift 3
out=gpurun_out/ncu
mkdir -p $out
ncu --set full --import-source on --clock-control none -k "regex:$k" -s "$skip" -c 1 -o $out/$tag -f \
    python bench.py "$@" --no-cpu-baseline > $out/$tag.log 2>&1
echo "$tag capture rc=$?"
ncu -i $out/$tag.ncu-rep --page raw --csv > $out/$tag.raw.csv 2>/dev/null
ncu -i $out/$tag.ncu-rep --page source --csv > $out/$tag.source.csv 2>/dev/null
[ -z "${KEEP_REP:-}" ] && rm -f $out/$tag.ncu-rep
ls -la $out | grep $tag
