mkdir -p gpurun_out/v8
timeout 500 python probes/svm_train.py 20000 > gpurun_out/v8/svm_train.log 2>&1; echo train rc=$?
timeout 300 python bench.py --workload svm_dual --cpu-iters 3 > gpurun_out/v8/bench_svm.jsonl 2> gpurun_out/v8/bench_svm.err; echo bsvm rc=$?
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/v8/t_svm_dual.csv python bench.py --workload svm_dual --steps 1 --warmup 3 --iters 50 --no-cpu-baseline > gpurun_out/v8/t_svm.log 2>&1; echo ncu1 rc=$?
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_slot_hess_sym -s 5 -c 1 -o gpurun_out/v8/full_svm_dual -f python bench.py --workload svm_dual --steps 1 --warmup 3 --iters 50 --no-cpu-baseline > gpurun_out/v8/full_svm.log 2>&1; echo ncu2 rc=$?
timeout 300 python bench.py > gpurun_out/v8/bench_cfg4.jsonl 2> gpurun_out/v8/bench_cfg4.err; echo cfg4 rc=$?
