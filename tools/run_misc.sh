cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for g in 444 443 296; do echo "grid $g"; NB_GRID_OVERRIDE=$g python tools/perf_quick.py C2 C3-f32; done > gpurun_out/grid_sweep.log 2>&1
python tools/perf_quick.py C3-f64 >> gpurun_out/grid_sweep.log 2>&1
