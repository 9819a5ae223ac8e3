for cfg in c2 c4 c5; do
for b in 512 1024; do for pre in 1 4; do
echo "== $cfg block=$b pre=$pre"
GT_LEVEL_BLOCK=$b GT_LEVEL_PRE=$pre python tools/gpu_probe.py $cfg --tasks wordcount,invertedindex,termvector --reps 3 2>&1 | grep -E "k_td_levels|wordcount|invertedindex|termvector"
done; done; done
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
