cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json; tail -2 gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 150 --warmup 10 --no-cpu-baseline --e2e-windows 1 --no-alternatives > /dev/null 2>&1
for k in assembled assembled_sym matrix_free; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 20 -c 1 -o gpurun_out/prof_c2_$k python bench.py --kernel $k --steps 30 --warmup 10 --no-cpu-baseline --e2e-windows 1 --no-alternatives > gpurun_out/ncu_$k.log 2>&1
tail -1 gpurun_out/ncu_$k.log
done
timeout 900 ncu --set full --clock-control none -k regex:k_step -s 5 -c 1 -o gpurun_out/prof_c4_assembled python bench.py --config c4 --kernel assembled --steps 10 --warmup 5 --no-cpu-baseline --e2e-windows 1 --no-alternatives > gpurun_out/ncu_c4.log 2>&1
tail -1 gpurun_out/ncu_c4.log
