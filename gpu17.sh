cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
free -g | head -2
timeout 1800 python bench.py --config c5 --kernel matrix_free --steps 50 --warmup 5 --no-cpu-baseline --no-alternatives --e2e-windows 1 --obs-every 50 > gpurun_out/bench_c5_mf.json 2> gpurun_out/bench_c5_mf.err
tail -1 gpurun_out/bench_c5_mf.json | cut -c1-1500; tail -3 gpurun_out/bench_c5_mf.err
