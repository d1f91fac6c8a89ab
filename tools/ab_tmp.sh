timeout 600 python -m pytest tests/test_gpu.py tests/test_gpu_dist.py -q -x 2>&1 | tail -1
for i in 1 2 3; do
for v in head cur; do
cp build/$v/libgtree_b200.so paper_2305_00645_b200/; timeout 120 python tools/probe.py c2 | cut -c1-30 | sed "s/^/$v /"
done
done
GT_COUNT_TS=1 GT_HC_TIMING=1 timeout 120 python tools/probe.py tl 2>/dev/null | head -3
