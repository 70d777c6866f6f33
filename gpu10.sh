cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for v in 0 1 3; do
  ENS_MF_VARIANT=$v timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline > gpurun_out/bench_mf_v$v.json 2>&1
  tail -1 gpurun_out/bench_mf_v$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mf v$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
for k in assembled assembled_sym matrix_free; do
  timeout 900 python bench.py --config c4 --kernel $k --no-cpu-baseline --steps 1000 --warmup 50 > gpurun_out/bench_c4_$k.json 2> gpurun_out/bench_c4_$k.err
  tail -1 gpurun_out/bench_c4_$k.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $k', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; tail -2 gpurun_out/bench_c4_$k.err
done
