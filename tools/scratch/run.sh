python tools/gpu_probe.py c2 c3 c4 c5 --reps 3 > gpurun_out/probe.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.txt 2>&1
