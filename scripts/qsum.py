import json, sys, glob
for f in sorted(glob.glob('gpurun_out/q_*.json')):
    try:
        d = json.load(open(f))
    except Exception:
        print(f, 'ERR'); continue
    top = sorted(d['kernels'].items(), key=lambda x: -x[1]['ms_per_step'])[:int(sys.argv[1]) if len(sys.argv) > 1 else 6]
    print('%-28s %.3f ms %.3f Ge/s  ' % (f[13:-5], d['ms_per_step'], d['value'] / 1e9) +
          ' '.join('%s=%.3f' % (k, v['ms_per_step']) for k, v in top))
