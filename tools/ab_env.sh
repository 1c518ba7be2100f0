#!/bin/bash
# A/B of an environment knob on the compress workload: median compress/decompress ms
# usage: tools/ab_env.sh "EBCC_X=1" "EBCC_X=0" [iters]
it=${3:-9}
for round in 1 2; do
for cfg in "$1" "$2"; do
  out=$(env $cfg python tools/prof_compress.py 37 $it 2>&1)
  echo "$cfg: $(echo "$out" | python -c "
import sys,re,statistics as s
t=sys.stdin.read()
c=[float(m) for m in re.findall(r'^compress wall ([0-9.]+)', t, re.M)][1:]
d=[float(m) for m in re.findall(r'^decompress wall ([0-9.]+)', t, re.M)][1:]
print('compress median %.2f min %.2f | decompress median %.2f min %.2f' % (s.median(c), min(c), s.median(d), min(d)))
")"
done
done
