tail -2 gpurun_out/gpu_tests.log
python - <<'P'
import json
for f in ['bench_c','bench_u','bench_c4_chung_lu','bench_c4_chung_lu_u','bench_c3_grid','bench_c3_grid_u']:
    try:
        d=json.load(open(f'gpurun_out/{f}.json'))
        print(f'{f:22s}', 'ms/step %.3f' % d['ms_per_step'], 'G/s %.2f' % (d['value']/1e9), 'decide ms %.3f' % d['roofline']['ms_per_iter'], 'frac %.3f' % d['roofline']['frac'])
    except Exception as e: print(f, 'ERR', e)
P
