cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1 2 3; do
  ENS_MF_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "matrix_free" > gpurun_out/pytest_mf$v.log 2>&1; tail -1 gpurun_out/pytest_mf$v.log
  ENS_MF_VARIANT=$v timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline > gpurun_out/bench_mf_v$v.json 2>&1
  tail -1 gpurun_out/bench_mf_v$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant $v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
ENS_A1_VEC4=1 timeout 300 python bench.py --kernel assembled --no-cpu-baseline > gpurun_out/bench_a1_vec4.json 2>&1
tail -1 gpurun_out/bench_a1_vec4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('a1 vec4', d['value'], d['ms_per_step'], d['roofline']['frac'])"
timeout 300 python bench.py --kernel assembled --no-cpu-baseline --n-s 128 > gpurun_out/bench_a1_128.json 2>&1
tail -1 gpurun_out/bench_a1_128.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('a1 ns128 vec2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
