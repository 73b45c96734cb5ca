tail -2 gpurun_out/gpu_tests.log
python - <<'P'
import json
for f in ['bench_c','bench_u']:
    try:
        d=json.load(open(f'gpurun_out/{f}.json'))
        print(f, 'ms/step %.3f' % d['ms_per_step'], 'decide ms %.3f' % d['roofline']['ms_per_iter'], 'e2e %.3f G/s' % (d['e2e']['value']/1e9))
    except Exception as e: print(f, 'ERR', e)
P
