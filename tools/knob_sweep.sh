# Fused-kernel experiment knobs (environment variables read by the launcher), FMA build,
# 256^3 O3 HLL: prints knob, G zone/s, kernel ms per launch. Usage: bash tools/knob_sweep.sh "ENV=.. ENV2=.." ...
for k in "$@"; do
  env $k python bench.py --steps 20 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$k', round(d['value']), round(d['roofline']['kernel_ms_per_launch'],4))"
done
