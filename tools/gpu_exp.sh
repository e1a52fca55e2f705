cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NB_SPLIT_MAX_N=100000 timeout 900 python -m pytest tests -m gpu -x -q -k "small_simulate or ragged or zero_softening or coincident or golden or c1 or full_size_trajectory_vs or uniform_mass or two_body" > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
timeout 900 python tools/small_n_bench.py 10 2048,4096,6144,8192,16384,32768 > gpurun_out/split_n.md 2>&1
