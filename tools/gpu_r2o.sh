#!/bin/bash
./tools/ex2_h2_bench | head -8
ncu --set full -k regex:k_ex -c 2 -o gpurun_out/ex2_probe ./tools/ex2_h2_bench > /dev/null 2>&1
ncu -i gpurun_out/ex2_probe.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin)); h = rows[0]
for k in h:
    if 'pipe_xu' in k and ('avg.pct' in k) or 'sm__cycles_active.avg' == k or k.startswith('gpu__time_duration.sum'):
        print(k, [r[h.index(k)] for r in rows[2:]])
"
