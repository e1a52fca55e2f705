cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "gravitational" > gpurun_out/pytest_g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g.log
