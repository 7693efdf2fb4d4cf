mkdir -p gpurun_out
./scripts/micro/fp64peak | tee gpurun_out/fp64peak.log
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/fp64peak.log') if l.startswith('{')]
d={r['op']+'_gops': r['gops'] for r in rows}
d['how']='scripts/micro/fp64peak.cu: 8 independent __dadd_rn / __dmul_rn chains per thread, 8 CTAs x 256 threads per SM, best of 5, CUDA events'
json.dump(d, open('profiles/r02_fp64_peak.json','w'), indent=1)
json.dump(d, open('gpurun_out/r02_fp64_peak.json','w'), indent=1)
print(d)
PY
CONFIGS="2" TAG=cfgsk bash scripts/gpu_configs.sh 2>&1 | cut -c1-200
tail -1 gpurun_out/cfgsk_cfg2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['roofline']))"
