# Same-call A/B of the working tree against HEAD on the GPU box (variant
# libraries prebuilt here by tools/ab_build.sh): alternates `probe.py c2`
# (and optionally `probe.py walk`) REPS times.
#   bash tools/ab_head.sh [REPS] [walk]
reps=${1:-3}
for i in $(seq $reps); do
  for v in head cur; do
    cp build/$v/libgtree_b200.so paper_2305_00645_b200/
    timeout 120 python tools/probe.py c2 | cut -c1-80 | sed "s/^/$v /"
  done
done
if [ "$2" = walk ]; then
  for v in head cur; do
    cp build/$v/libgtree_b200.so paper_2305_00645_b200/; timeout 200 python tools/probe.py walk | sed "s/^/$v /"
  done
fi
cp build/cur/libgtree_b200.so paper_2305_00645_b200/
