# Bench lines of the other workloads (profiles/r2_variants.jsonl): configs[0] (C1), O2 / O4 at
# 256^3, O3 / O2 at 384^3 (C3 proxies) and 512^3 (configs[4] on one GPU), MHD 384^3, CED 256^3,
# the formally fourth-order ADER step at 256^3, the RK2 / RK3 integrators (the paper's CFD RK row).
# No CPU baseline (the headline has it).
set -e
mkdir -p gpurun_out
out=gpurun_out/variants.jsonl; : > $out
for a in "--workload c1" "--order 2" "--order 4" "--n 384" "--n 384 --order 2" "--n 512" "--n 512 --order 2" "--workload mhd" "--workload ced" "--workload ader4" "--integrator rk2 --order 2" "--integrator rk3 --order 3" "--workload mhd --order 4" "--workload ced --order 4" "--workload mhd --mhd-hlld"; do
  python bench.py $a --no-cpu-baseline --e2e-steps 2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['args']='$a'; print(json.dumps(d))" >> $out
done
python - <<'P'
import json
for l in open("gpurun_out/variants.jsonl"):
    d = json.loads(l)
    ob = d.get("other_build") or {}
    print(d["args"], round(d["value"]), "other", round(ob.get("value", 0)), "frac", round((d.get("roofline") or {}).get("frac", 0), 3))
P
