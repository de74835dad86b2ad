# compute-sanitizer over the kernels added late in round 2: the in-kernel halo stores (seam
# kernels with the peer-store switch, the ring path's plane copy) on 2 / 4 slabs of one GPU,
# the single-launch ghost fill and the folded advance (configs[0]-sized stepper, graph replay),
# the rewritten MHD / CED order-4 predictors. Run on the GPU box.
mkdir -p gpurun_out
out=gpurun_out/r2c_sanitizer.txt; : > $out
for tool in memcheck racecheck synccheck; do
  for t in "tests/test_domain_gpu.py -k \"peer_store and (shape0-0-True or shape1-3-False or shape0-3-False)\"" \
           "tests/test_gpu_parity.py -k graph" \
           "tests/test_seam_gpu.py -k configs0" \
           "tests/test_mhd4_gpu.py -k conserves" \
           "tests/test_ced4_gpu.py -k \"relaxation_accuracy and 5.0\""; do
    r=$(eval timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest -q -p no:cacheprovider $t 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY" | tr '\n' ' ')
    echo "$tool | $t | $r" >> $out
  done
done
cat $out
