# Round-2 measurement set: FP32 peak, bench lines for every config, the
# reference arm, per-launch lists (north_star, C, E) -> gpurun_out/r2/
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv,noheader
./tools/micro/fp32_peak | tee gpurun_out/r2/fp32_peak.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2/bench_north_star.json 2> gpurun_out/r2/bench_north_star.err
for c in A B C D E; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2/bench_$c.json 2>gpurun_out/r2/bench_$c.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r2/bench_reference.json 2>/dev/null
for c in north_star B C E; do bash tools/ncu_launches.sh $c r2/launches_$c > gpurun_out/r2/launches_$c.txt; done
for f in gpurun_out/r2/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline',{}); e=d.get('e2e',{})
print('$f'.split('/')[-1], round(d.get('ms_per_step',0),3), {k:round(v,3) for k,v in d.get('breakdown_ms',{}).items()}, 'frac', r.get('frac') and round(r['frac'],3), 'e2e_ms', e.get('ms_per_step') and round(e['ms_per_step'],2))" 2>/dev/null; done
cat gpurun_out/r2/launches_north_star.txt
