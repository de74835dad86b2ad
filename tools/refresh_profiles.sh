# Headline evidence in one gpurun call: bench line, ncu --set full of one fused launch (FMA and
# bit-exact builds, 256^3 O3 HLL), the serialised launch list of the timed steps.
# Usage: gpurun -- 'bash tools/refresh_profiles.sh'; then profiles/summarize.py locally.
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_o3_256.json 2> gpurun_out/bench.err
for b in fma exact; do
  flag=""; [ $b = exact ] && flag="--exact"
  ncu --set full --import-source on --clock-control none -k regex:fused_ader -s 3 -c 1 \
      -o gpurun_out/fused_o3_256_$b -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
      --only-timed $flag > gpurun_out/ncu_$b.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_o3_256_fma.csv python bench.py --steps 5 --warmup 3 \
    --no-cpu-baseline --only-timed > gpurun_out/launches.log 2>&1
tail -c 600 gpurun_out/bench_o3_256.json
