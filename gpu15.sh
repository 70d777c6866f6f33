cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ENS_MF_VARIANT=6 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "matrix_free and (spmm or equivalence)" > gpurun_out/pytest_v6.log 2>&1; tail -2 gpurun_out/pytest_v6.log
for ns in 64 128; do
  ENS_MF_VARIANT=6 timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline --no-alternatives --n-s $ns > gpurun_out/bench_mf_v6_$ns.json 2>&1
  tail -1 gpurun_out/bench_mf_v6_$ns.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mf v6 ns $ns', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
