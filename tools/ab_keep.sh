#!/bin/bash
# A/B of the rows of A p kept in registers by cg_tile_kernel (HIVC_CG_KEEP30/23/15), rebuilt on the box per arm.
# Per arm: 1080p / 540p single-solve times (tools/level_time.py, cg_trace phases of CTA 0) and two bench runs.
arm() {
  touch paper_2008_10273_b200/csrc/cg_tile.cuh
  HIVC_NVCC_EXTRA="-DHIVC_CG_KEEP30=$1 -DHIVC_CG_KEEP23=$2 -DHIVC_CG_KEEP15=$3" python -m paper_2008_10273_b200.build > /dev/null 2>&1 || { echo "build failed $*"; return; }
  echo "== keep30=$1 keep23=$2 keep15=$3"
  python tools/level_time.py 2>/dev/null | tail -2
  HIVC_DEBUG=cg_trace python tools/level_time.py 1080x1920 2>&1 | grep -i "phase\|us" | tail -4
  for i in 1 2; do python bench.py --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', round(d['ms_per_step'],2), round(d['value']), round(d['e2e']['value']), 'tile_us', round(d['roofline']['avg_launch_us']))"; done
}
arm 0 0 0
arm 14 16 15
arm 16 23 15
arm 8 16 15
arm 20 23 15
arm 0 0 0
arm 14 16 15
