# executor knob sweep on the C2 bench: one bench run per JSON request override (argv, or the default list)
set -u
if [ $# -gt 0 ]; then list=("$@"); else list=('{}' '{"opt_priority": true}'); fi
for j in "${list[@]}"; do
  echo "== $j"
  HY_DEBUG_ARENA=1 timeout 200 python bench.py --steps 2 --warmup 3 --no-variants --no-cpu-baseline ${OPT_STATE:+--opt-state $OPT_STATE} --exec-json "$j" 2>&1 | grep -E "arena dev|^\{|Error|error" | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); sr=d['shard_roofline']; b=d['bytes_per_step']
        print(d['value'], sr['achieved_h2d_GBps'], sr.get('actual_bytes_link_frac'), 'param_h2d', b['param_h2d_bytes_per_pass']/1e9, 'wb', b['writeback_d2h_bytes_per_pass']/1e9)
    else: print(l.strip())
"
done
