cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
tail -8 gpurun_out/pytest_gpu.log
for k in assembled assembled_sym matrix_free; do
  timeout 300 python bench.py --kernel $k --no-cpu-baseline > gpurun_out/bench_$k.json 2>&1
  tail -1 gpurun_out/bench_$k.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'], d['clocks']['sm_mhz'], d['e2e']['value'])"
  timeout 300 python bench.py --kernel $k --no-cpu-baseline --n-s 128 > gpurun_out/bench_${k}_128.json 2>&1
  tail -1 gpurun_out/bench_${k}_128.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k ns128', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_assembled_sym -s 20 -c 1 -o gpurun_out/prof_a1s python bench.py --kernel assembled_sym --steps 30 --warmup 10 --no-cpu-baseline --e2e-windows 1 > gpurun_out/ncu_a1s.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_matrix_free -s 20 -c 1 -o gpurun_out/prof_a2v3 python bench.py --kernel matrix_free --steps 30 --warmup 10 --no-cpu-baseline --e2e-windows 1 > gpurun_out/ncu_a2.log 2>&1
tail -1 gpurun_out/ncu_a2.log
