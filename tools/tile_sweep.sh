# tile-shape sweep of the fused kernel (HC_TUNE=1 build): O3 and O2, FMA build, 256^3
for o in 3 2; do for c in 1 2 3 4 5; do
  HC_FUSED_CFG=$c python bench.py --order $o --steps 10 --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('O$o cfg', $c, round(d['value']), round(d['roofline']['kernel_ms_per_launch'],3))"
done; done
