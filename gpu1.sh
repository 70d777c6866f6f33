set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -2 gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline > gpurun_out/bench_a2.json 2> gpurun_out/bench_a2.err
cat gpurun_out/bench_a2.json; tail -3 gpurun_out/bench_a2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 50 --warmup 10 --no-cpu-baseline --e2e-windows 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_assembled -s 20 -c 2 -o gpurun_out/prof_a1 python bench.py --steps 30 --warmup 10 --no-cpu-baseline --e2e-windows 1 > gpurun_out/ncu_a1.log 2>&1
tail -3 gpurun_out/ncu_a1.log
