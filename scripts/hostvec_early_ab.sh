#!/bin/bash
# A/B on one box: the hostvec copy-in grid launched as a programmatic
# dependent of the stream's previous kernel (KBLAS_HOSTVEC_EARLY=1, default)
# or the ordinary way (0).  Queued and one-at-a-time numpy-vector calls
# (scripts/queue_overhead.py) and the bench's configs[0] block.
O=${1:-gpurun_out/hostvec_early_ab.log}
: > $O
for rep in 1 2; do
  for early in 0 1; do
    echo "=== KBLAS_HOSTVEC_EARLY=$early rep $rep" >> $O
    KBLAS_HOSTVEC_EARLY=$early timeout 300 python scripts/queue_overhead.py 2>&1 | grep -E "^n=|us/call" >> $O
    KBLAS_HOSTVEC_EARLY=$early timeout 300 python bench.py --op dgemv --n 4096 --steps 200 --no-cpu 2>/dev/null \
      | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.readline()); e=d['e2e']; print('bench cfg0 value', d['value'], 'e2e', e['value'], 'queued', e['queued']['value'])" >> $O
  done
done
cat $O
