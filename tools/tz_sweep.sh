# planes-per-chunk sweep of the fused kernel (256^3 O3, FMA and exact builds)
for tz in 24 32 43 52 64 86 128 auto; do
  for f in "--fast" ""; do
    if [ $tz = auto ]; then unset HC_TZ; else export HC_TZ=$tz; fi
    python bench.py --steps 10 --no-cpu-baseline --e2e-steps 1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tz', '$tz', d['config']['build'], round(d['value']), round(d['roofline']['kernel_ms_per_launch'],3))"
  done
done
