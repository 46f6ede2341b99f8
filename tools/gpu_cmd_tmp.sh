mkdir -p gpurun_out
timeout 2400 python tools/dc_sweep.py 2 > gpurun_out/dc_sweep.jsonl 2> gpurun_out/dc_sweep.err
python -c "
import json
for l in open('gpurun_out/dc_sweep.jsonl'):
    d=json.loads(l); print(d['family'], d['level'], d['n'], d['eps'], 'dc' if d['dc'] else 'nodc', d.get('pcg_iters'), d.get('gmres_iters'), round(d.get('t_factor_s',0),3), d.get('error','')[:60])
"
tail -3 gpurun_out/dc_sweep.err
