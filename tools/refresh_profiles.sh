# Headline evidence in one gpurun call: the bench line; ncu --set full of one step's compute
# launches in both builds (the seam kernel pair: seam_ader_kernel + seam_fix_kernel; the
# bit-exact build's pair keeps the reference's association) at 256^3 O3 HLL; the serialised launch list of the
# timed steps. The captures are summarised on the box (profiles/summarize.py -> gpurun_out/
# r2_*.json) and the .ncu-rep files dropped so the results fit the 64 MiB copy-back.
# Usage: gpurun -- 'bash tools/refresh_profiles.sh'; copy gpurun_out/r2_*.json to profiles/.
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_o3_256.json 2> gpurun_out/bench.err
ncu --set full --import-source on --clock-control none -k regex:seam_ -s 8 -c 2 \
    -o /tmp/fused_o3_256_fma -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --only-timed > gpurun_out/ncu_fma.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:seam_ -s 8 -c 2 \
    -o /tmp/fused_o3_256_exact -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --only-timed --exact > gpurun_out/ncu_exact.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches_o3_256_fma.csv python bench.py --steps 5 --warmup 3 \
    --no-cpu-baseline --only-timed > gpurun_out/launches.log 2>&1
python profiles/summarize.py /tmp/fused_o3_256_fma.ncu-rep r2_fused_o3_256_fma \
    --launches gpurun_out/r2_launches_o3_256_fma.csv --zones 16777216 > /dev/null
python profiles/summarize.py /tmp/fused_o3_256_exact.ncu-rep r2_fused_o3_256_exact \
    --zones 16777216 > /dev/null
cp profiles/r2_fused_o3_256_fma.json profiles/r2_fused_o3_256_exact.json gpurun_out/
ncu -i /tmp/fused_o3_256_fma.ncu-rep --page source --csv --print-source sass \
    -k regex:seam_ader > gpurun_out/r2_seam_ader_sass.csv 2>/dev/null || true
gzip -f gpurun_out/r2_seam_ader_sass.csv || true
tail -c 600 gpurun_out/bench_o3_256.json
