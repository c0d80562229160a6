import json, sys
hdr = ""
for ln in open(sys.argv[1]):
    if ln.startswith('env'): hdr = ln.strip(); continue
    if not ln.startswith('{'): print(ln[:300].rstrip()); continue
    d = json.loads(ln); c = d['costs']
    print(hdr, 'cl', d['cluster'], 'ms %.2f' % d['ms'], 'pcg_it', c[-1][2], 'pcg_ms', d['prof'].get('pcg'),
          'us/it %.1f' % (1000 * d['prof'].get('pcg', 0) / max(c[-1][2], 1)),
          'inv', d['prof'].get('coarse_inverse'), 'final %.10g' % c[-1][0])
