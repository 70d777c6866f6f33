cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -k "stress" > gpurun_out/pytest_stress.log 2>&1; tail -15 gpurun_out/pytest_stress.log
