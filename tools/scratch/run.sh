python tools/gpu_probe.py c2 c3 c4 c5 --tasks wordcount --pinned --reps 3 > gpurun_out/probe_open.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.txt 2>&1
compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "long_records or composed_all_tasks and c2-0.002" > gpurun_out/memcheck_chain.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_chain.txt
