set -x
nvidia-smi; nproc; lscpu | head -25; free -g; python -c "import torch;print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_probe.csv &
CP=$!
./tools/pipe_peaks
./tools/pipe_peaks
kill $CP
