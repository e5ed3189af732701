#!/bin/bash
# every BASELINE config on one B200 (DESIGN.md section 8 table); steps kept
# below each config's iterations to convergence (the timed FastPAM1 steps are
# one queued kmedoids_swap_iters call)
cd $GRAFT_REPO_ROOT
for spec in "1 fastpam1 1 2" "2 fastpam1 3 5" "3 fastpam1 5 30" "3 fastpam2 3 10" "4 fastpam1 5 40" "5 fastpam1 3 20" "5 fastpam2 3 10"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --variant $2 --warmup $3 --steps $4 --no-fasterpam --no-dissimilarity --no-clara --cpu-seconds 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; e=d.get('e2e') or {}; c=d.get('cpu_baseline') or {}
print('C$1 $2', 'ms/step %.4f' % d['ms_per_step'], 'pairs/s %.3e' % d['value'], 'stream %.4f' % r['kernel_ms'], 'frac_copy %.3f' % r['frac'], 'frac_read %.3f' % r.get('frac_of_read_only_peak', 0), 'e2e %.3e' % e.get('value', 0), 'e2e_s %.3f' % e.get('seconds', 0), 'jobs', e.get('jobs_s'), 'cpu %.3e' % c.get('value', 0), 'init %s' % d['init'], flush=True)"
done
