# compute-sanitizer (memcheck, racecheck, synccheck) over the round-2 kernels: the seam pair in
# both builds (tests/test_seam_gpu.py vs_reference on 3 meshes: FMA vs the restatement's
# tolerance, exact bitwise), the order-4 predictor (uniform state + conservation), the MHD
# HLLD face solver (bitwise vs the restatement, random 3D data). Run on the GPU box.
mkdir -p gpurun_out
out=gpurun_out/r2b_sanitizer.txt; : > $out
SEL_SEAM='vs_reference and (shape0 or shape1 or shape8)'
for tool in memcheck racecheck synccheck; do
  for t in "tests/test_seam_gpu.py -k \"$SEL_SEAM\"" \
           "tests/test_ader4_gpu.py -k \"uniform or conserves\"" \
           "tests/test_mhd_gpu.py -k \"bitwise and random and 1]\""; do
    r=$(eval timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest -q -p no:cacheprovider $t 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY" | tr '\n' ' ')
    echo "$tool | $t | $r" >> $out
  done
done
cat $out
