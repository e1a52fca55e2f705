cd $GRAFT_REPO_ROOT
NB_LIB_PATH=$PWD/paper_2203_08263_b200/libnbody_b200_check.so timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_checked.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_checked.log
NB_LIB_PATH=$PWD/paper_2203_08263_b200/libnbody_b200_check.so python tools/sanitize_case.py >> gpurun_out/pytest_gpu_checked.log 2>&1
