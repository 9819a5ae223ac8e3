python -m pytest tests -m gpu -x -q > gpurun_out/gputests.txt 2>&1
python tools/gpu_probe.py c2 c3 c4 c5 --pinned --reps 3 --top 10 > gpurun_out/probe_all.txt 2>&1
