# A/B of the lane kernels' register cap (GT_LANE_MINB) on the GPU box
for mb in 1 3 4; do
  touch paper_2305_00645_b200/csrc/*.cu
  make -s -j8 NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DGT_LANE_MINB=$mb" paper_2305_00645_b200/libgtree_b200.so > /dev/null 2>&1
  echo "== GT_LANE_MINB=$mb"
  timeout 200 python tools/quick_time.py 2>&1 | grep -E "per-kernel|infer|train ms"
done
