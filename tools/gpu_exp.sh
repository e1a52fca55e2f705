cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NB_LIB_PATH=$GRAFT_REPO_ROOT/paper_2203_08263_b200/libnbody_b200_check.so timeout 1500 python -m pytest tests -m gpu -q -x -k "small_simulate or ragged or c1 or golden or zero_softening or coincident or persistent or single_body or two_body" > gpurun_out/pytest_check.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_check.log
