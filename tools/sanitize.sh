#!/bin/bash
# compute-sanitizer tiers over the device path (run on the GPU box):
#   memcheck + racecheck + synccheck on the gadget parity tests (width 64) and
#   on smoke() (the C1 SPECT-shaped depth-4 tree + inference, checked
#   share-for-share against the oracle).  Logs land in gpurun_out/.
set -u
out=${1:-gpurun_out}
mkdir -p "$out"
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
for tool in memcheck racecheck synccheck; do
  $CS --tool $tool --log-file "$out/sanitize_${tool}_gadgets.log" \
    python -m pytest tests/test_gpu.py -x -q -p no:cacheprovider \
      -k "test_gadgets_share_exact_vs_oracle and 64 or test_division_argmin_oaa_kats" > "$out/sanitize_${tool}_gadgets.out" 2>&1
  echo "$tool gadgets rc=$?"
  $CS --tool $tool --log-file "$out/sanitize_${tool}_c1.log" \
    python -c "import __graft_entry__ as g; g.smoke()" > "$out/sanitize_${tool}_c1.out" 2>&1
  echo "$tool c1 rc=$?"
done
# the fused count (paired x-plane copies), early oaa lanes, split partition (hybrid last partition) on a small depth-7 C2-shaped tree
for tool in memcheck racecheck synccheck; do
  $CS --tool $tool --log-file "$out/sanitize_${tool}_small_fused.log" \
    python tools/probe.py small > "$out/sanitize_${tool}_small_fused.out" 2>&1
  echo "$tool small_fused rc=$?"
done
# the full C2 tree (memcheck only: racecheck over ~120 launches of this size takes too long)
$CS --tool memcheck --log-file "$out/sanitize_memcheck_c2_tree.log" python tools/probe.py c2eager \
  > "$out/sanitize_memcheck_c2_tree.out" 2>&1
echo "memcheck c2_tree rc=$?"
