# Build the library with extra nvcc flags into build/<name>/libgtree_b200.so (A/B of compile-time switches):
#   bash tools/build_variant.sh NAME [nvcc flags ...]
# on the GPU box: cp build/NAME/libgtree_b200.so paper_2305_00645_b200/ before the run.
set -e
name=$1; shift
out=build/$name; mkdir -p $out
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for f in gt_gadget_api gt_train gt_infer gt_party; do
  nvcc $FL "$@" -c paper_2305_00645_b200/csrc/$f.cu -o $out/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libgtree_b200.so $out/*.o -lcudart
