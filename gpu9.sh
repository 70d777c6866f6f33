cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for rows in 64 16 8; do
for ns in 64 128; do
  ENS_MF_ROWS=$rows timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline --n-s $ns > gpurun_out/bench_mf_${rows}_$ns.json 2>&1
  tail -1 gpurun_out/bench_mf_${rows}_$ns.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mf rows $rows ns $ns', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_matrix_free -s 20 -c 1 -o gpurun_out/prof_a2v6 python bench.py --kernel matrix_free --steps 30 --warmup 10 --no-cpu-baseline --e2e-windows 1 > gpurun_out/ncu_a2.log 2>&1
tail -1 gpurun_out/ncu_a2.log
