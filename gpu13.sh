cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -k "c3 or c4" > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for h in 0 1 2; do
  ENS_A1S_HINTS=$h timeout 300 python bench.py --kernel assembled_sym --no-cpu-baseline --no-alternatives > gpurun_out/bench_a1s_h$h.json 2>&1
  tail -1 gpurun_out/bench_a1s_h$h.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('a1s hint $h', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
ENS_A1S_HINTS=1 timeout 900 ncu --set full --clock-control none -k regex:k_step -s 20 -c 1 -o gpurun_out/prof_a1s_h1 python bench.py --kernel assembled_sym --steps 30 --warmup 10 --no-cpu-baseline --e2e-windows 1 --no-alternatives > gpurun_out/ncu_a1s.log 2>&1
tail -1 gpurun_out/ncu_a1s.log
