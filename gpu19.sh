cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ENS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo "rc=$?"; cat gpurun_out/bench_2rank.json | cut -c1-600; tail -3 gpurun_out/bench_2rank.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 5 --warmup 1 > gpurun_out/bench_ref_2rank.json 2> gpurun_out/bench_ref_2rank.err
echo "rc=$?"; cat gpurun_out/bench_ref_2rank.json | cut -c1-300; tail -3 gpurun_out/bench_ref_2rank.err
