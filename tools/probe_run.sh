nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/fp64_probe.bin > gpurun_out/fp64_probe.txt 2>&1
python tools/probe_host.py > gpurun_out/probe_host.json 2>&1
kill $SMI
nvidia-smi -q | head -60 > gpurun_out/smi.txt
