#!/bin/bash
# CTA rasterisation groups (HLF_RASTER = G y rows per group; 0 = x-fastest):
# step time and DRAM bytes per cell of the three 3D m = 3 launches at 512x512x256.
# usage (GPU box): tools/raster_sweep.sh "0 4 8 16" > out.txt
for g in ${1:-0 4 8 16}; do
  echo "G=$g $(HLF_RASTER=$g python tools/time_kernel.py 3 3 512x512x256 10)"
  HLF_RASTER=$g ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tiled3d \
    --launch-skip 6 --launch-count 3 --csv python tools/time_kernel.py 3 3 512x512x256 1 2>/dev/null |
    python3 -c "
import csv, sys
rows = list(csv.reader([l for l in sys.stdin if l.startswith('\"')]))
h = rows[0]; acc = {}
for r in rows[1:]:
    k = r[h.index('Kernel Name')].split('tiled3d<')[-1].split('>')[0]
    acc.setdefault(k, 0.0); v = float(r[h.index('Metric Value')].replace(',', ''))
    u = r[h.index('Metric Unit')]; acc[k] += v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
cells = 512 * 512 * 256
print('   DRAM B/cell', {k: round(v / cells) for k, v in acc.items()})
"
done
