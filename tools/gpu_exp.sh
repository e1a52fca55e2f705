cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "exchange or sharded or multi_rank or peer or symmetric" > gpurun_out/pytest_comm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_comm.log
