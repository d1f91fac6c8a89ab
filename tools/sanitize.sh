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
