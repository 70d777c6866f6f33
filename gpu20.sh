cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf -k "reassembl" > gpurun_out/pytest_re.log 2>&1; tail -15 gpurun_out/pytest_re.log
