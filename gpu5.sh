cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
tail -8 gpurun_out/pytest_gpu.log
ENS_A1_VEC4=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "spmm_parity or equivalence" > gpurun_out/pytest_vec4.log 2>&1; tail -2 gpurun_out/pytest_vec4.log
for v in 0 1 2 3; do
  ENS_MF_VARIANT=$v timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline > gpurun_out/bench_mf_v$v.json 2>&1
  tail -1 gpurun_out/bench_mf_v$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mf variant $v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
for pf in 0 1; do
ENS_A1_PREFETCH=$pf timeout 300 python bench.py --kernel assembled --no-cpu-baseline > gpurun_out/bench_a1_pf$pf.json 2>&1
tail -1 gpurun_out/bench_a1_pf$pf.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('a1 prefetch $pf', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
