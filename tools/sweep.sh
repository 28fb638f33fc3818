# Config 3/4/5 sweep on one B200: one bench line per workload x dtype.
out=gpurun_out/sweep.jsonl
: > $out
for w in bigbird_like bart_step longformer_like phi4_like qwen_audio_like biogpt_like blenderbot_like flan_t5_like pegasus_like moe_minicpm_like; do
  for d in bf16 fp32; do
    timeout 600 python bench.py --workload $w --dtype $d --steps 100 --warmup 10 2>/dev/null >> $out || echo "{\"workload\": \"$w\", \"dtype\": \"$d\", \"error\": true}" >> $out
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep.jsonl"):
    d = json.loads(l)
    if "error" in d: print(d); continue
    print(d["config"]["workload"][:40], d["dtype"], "p50 %.3f ms" % d["p50_ms"], "%.0f samples/s" % d["value"],
          "e2e %.0f" % d["e2e"]["value"], "cpu %.1f" % d.get("cpu_baseline", {}).get("value", 0), d["mode"], d["host_syncs_per_forward"],
          "frac %.2f" % (d["roofline"] or {}).get("frac", 0))
PY
