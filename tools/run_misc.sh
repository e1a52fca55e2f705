cd $GRAFT_REPO_ROOT
python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/sanitize_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.log
