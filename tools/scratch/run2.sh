GT_TRACE=2 python tools/gpu_probe.py c2 --tasks wordcount --pinned --reps 2 > gpurun_out/trace_c2.txt 2>&1
python tools/gpu_probe.py c2 c3 --tasks wordcount,invertedindex --pinned --reps 3 > gpurun_out/probe_open.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.txt 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
