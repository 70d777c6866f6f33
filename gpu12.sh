cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -k "matrix_free" > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for v in 0 1; do
for ns in 64 128; do
  ENS_MF_VARIANT=$v timeout 300 python bench.py --kernel matrix_free --no-cpu-baseline --no-alternatives --n-s $ns > gpurun_out/bench_mf_v${v}_$ns.json 2>&1
  tail -1 gpurun_out/bench_mf_v${v}_$ns.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mf v$v ns $ns', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 20 -c 1 -o gpurun_out/prof_c2_mf_ns python bench.py --kernel matrix_free --steps 30 --warmup 10 --no-cpu-baseline --e2e-windows 1 --no-alternatives > gpurun_out/ncu_mf.log 2>&1
tail -1 gpurun_out/ncu_mf.log
