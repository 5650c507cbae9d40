#!/bin/bash
# Build + bench several backward-kernel launch shapes (threads, LDGSTS stages, min CTAs/SM).
for cfg in ${CFGS:-"256 3 2" "256 4 1" "128 6 2" "128 4 3" "128 5 2" "256 5 1"}; do
  set -- $cfg
  QFS_NVCC_DEFINES="-DQFS_BWD_THREADS=$1 -DQFS_BWD_STAGES=$2 -DQFS_BWD_MINB=$3" python -c "from paper_2405_12866_b200 import build; build.build(force=True)" || continue
  python bench.py --steps 10 --no-cpu-baseline --no-tts 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$cfg', round(d['value']), round(d['ms_per_step'],3), r['avg_launch_us'], {k:round(v['ms']/v['launches']*1e3,2) for k,v in r['kernels'].items()})"
done
