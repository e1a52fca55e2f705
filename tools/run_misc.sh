cd $GRAFT_REPO_ROOT
for c in C3-f64 C2; do
python tools/profile_step.py $c 3 > gpurun_out/plain_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o gpurun_out/prof_$c python tools/profile_step.py $c 2 > gpurun_out/ncu_full_$c.log 2>&1
done
