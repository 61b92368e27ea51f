timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/ns_final.json 2> gpurun_out/ns_final.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ref_final.json 2> /dev/null
python - <<'PY'
import json
a = json.loads(open("gpurun_out/ns_final.json").read().strip().splitlines()[-1])
b = json.loads(open("gpurun_out/ref_final.json").read().strip().splitlines()[-1])
print("same_config", a["config"] == b["config"])
print(a["ms_per_step"], a["breakdown_ms"], a["e2e"]["ms_per_step"], a["clocks"], a["gpu_launches"])
print(b["ms_per_step"], b["value"])
PY
