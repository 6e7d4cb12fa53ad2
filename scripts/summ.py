import json, sys
for f in sys.argv[1:]:
    try:
        lines = [l for l in open(f) if l.startswith('{')]
        d = json.loads(lines[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    print(f, 'val %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'e2e %.3g' % d['e2e']['value'], 'launches', d.get('gpu_launches'))
    if 'roofline_kernels' in d:
        print('   kern', [(k['label'], round(k['launch_ms'], 4), round(k['frac'], 3)) for k in d['roofline_kernels']],
              'opTF %.0f' % d['roofline_operator']['achieved'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
