timeout 300 python tools/measure_tf32_peak.py gpurun_out/tf32_peak.json > gpurun_out/tf32.log 2>&1
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv >> gpurun_out/tf32.log
