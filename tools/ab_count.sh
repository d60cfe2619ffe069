#!/bin/bash
# A/B of count-kernel build variants (libtpgen_<v>.so, see build.py --variant): config 3 and 5 count mode
for v in "$@"; do
  if [ "$v" = base ]; then unset TPGEN_LIB_VARIANT; else export TPGEN_LIB_VARIANT=$v; fi
  echo "== $v"
  timeout 300 python tools/count_bench.py 2>&1 | python -c "
import sys, json
for line in sys.stdin:
    try: d = json.loads(line)
    except Exception: print(line.strip()); continue
    print(d['workload'], 'digest' if d['digest'] else 'nodig', 'dfs', d['ms_dfs'][-1], 'dev', d['ms_device'][-1], d['hash'][0] % 1000)
"
done
