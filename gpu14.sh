cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 1 4 5; do
  ENS_MF_VARIANT=$v timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline --no-alternatives > gpurun_out/bench_mf_v$v.json 2>&1
  tail -1 gpurun_out/bench_mf_v$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mf v$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['read_stream_GBs'], d['clocks']['sm_mhz'])"
done
