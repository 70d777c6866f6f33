cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
for k in assembled matrix_free; do
  timeout 300 python bench.py --kernel $k --no-cpu-baseline > gpurun_out/bench_$k.json 2> gpurun_out/bench_$k.err
  cat gpurun_out/bench_$k.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['kernel'], d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"; tail -2 gpurun_out/bench_$k.err
  ENS_GRAPH_STEPS=0 timeout 300 python bench.py --kernel $k --no-cpu-baseline > gpurun_out/bench_${k}_nograph.json 2>&1
  cat gpurun_out/bench_${k}_nograph.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nograph', d['config']['kernel'], d['value'], d['ms_per_step'])"
done
timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline --n-s 128 > gpurun_out/bench_mf128.json 2>&1; tail -1 gpurun_out/bench_mf128.json | cut -c1-400
timeout 300 python bench.py --kernel assembled --no-cpu-baseline --n-s 128 > gpurun_out/bench_a1128.json 2>&1; tail -1 gpurun_out/bench_a1128.json | cut -c1-400
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_matrix_free -s 20 -c 1 -o gpurun_out/prof_a2v2 python bench.py --kernel matrix_free --steps 30 --warmup 10 --no-cpu-baseline --e2e-windows 1 > gpurun_out/ncu_a2.log 2>&1
tail -2 gpurun_out/ncu_a2.log
