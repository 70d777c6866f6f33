cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline > gpurun_out/bench_a2.json 2> gpurun_out/bench_a2.err
cat gpurun_out/bench_a2.json; tail -3 gpurun_out/bench_a2.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 80 --csv --log-file gpurun_out/launches.csv python bench.py --steps 50 --warmup 10 --no-cpu-baseline --e2e-windows 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_matrix_free -s 20 -c 1 -o gpurun_out/prof_a2 python bench.py --kernel matrix_free --steps 30 --warmup 10 --no-cpu-baseline --e2e-windows 1 > gpurun_out/ncu_a2.log 2>&1
tail -2 gpurun_out/ncu_a2.log
