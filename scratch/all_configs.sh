#!/bin/bash
cd $GRAFT_REPO_ROOT
for spec in "1 fastpam1" "2 fastpam1" "3 fastpam1" "3 fastpam2" "4 fastpam1" "5 fastpam1" "5 fastpam2"; do
  set -- $spec
  timeout 400 python bench.py --config $1 --variant $2 --steps 30 --warmup 5 --no-fasterpam --no-dissimilarity --cpu-seconds 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; e=d.get('e2e') or {}; c=d.get('cpu_baseline') or {}
print('C$1 $2', 'ms/step %.4f' % d['ms_per_step'], 'pairs/s %.3e' % d['value'], 'stream %.4f' % r['kernel_ms'], 'frac_copy %.3f' % r['frac'], 'frac_read %.3f' % r.get('frac_of_read_only_peak', 0), 'e2e %.3e' % e.get('value', 0), 'e2e_s %.3f' % e.get('seconds', 0), 'cpu %.3e' % c.get('value', 0), 'init %s' % d['init'], flush=True)"
done
