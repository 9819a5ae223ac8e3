python tools/gpu_probe.py c2 c3 c4 c5 --pinned --reps 3 > gpurun_out/probe_all.txt 2>&1
