# bench lines for the main workloads (bash tools/gpu/r2_bench.sh [tag])
mkdir -p gpurun_out
t=${1:-x}
: > gpurun_out/bench_$t.jsonl
for w in "cfg3" "cfg3 --batch 64" "cfg3 --batch 8" "cfg3 --batch 1" "cfg4" "cfg1" "cfg2"; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log >> gpurun_out/bench_$t.jsonl
done
python - $t <<'PY'
import json,sys
for l in open("gpurun_out/bench_%s.jsonl" % (sys.argv[1] if len(sys.argv)>1 else "x")):
    try: j=json.loads(l)
    except Exception: print("BAD", l[:200]); continue
    print(j["config"]["workload"][:12], j["config"].get("global_batch"), "ms/step", j["ms_per_step"], "e2e", round(j["e2e"]["value"]), "kfrac", j["roofline"]["frac"], "stepfrac", j["step_roofline"]["frac"], "stages", {k: round(v,1) for k,v in j["stage_us_per_step"].items()}, "recall", j.get("recall_at_k"))
PY
