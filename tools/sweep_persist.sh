#!/bin/bash
for cfg in "256 4 1" "256 3 2" "128 5 2" "128 4 3"; do
  set -- $cfg
  QFS_NVCC_DEFINES="-DQFS_BWD_THREADS=$1 -DQFS_BWD_STAGES=$2 -DQFS_BWD_MINB=$3" python -c "from paper_2405_12866_b200 import build; build.build(force=True)" || continue
  for env in "QFS_PERSISTENT=0" "QFS_PERSISTENT=1 QFS_STAGGER=0" "QFS_PERSISTENT=1 QFS_STAGGER=1"; do
    env $env python bench.py --steps 10 --no-cpu-baseline --no-tts 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$cfg', '$env', round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms']/v['launches']*1e3,2) for k,v in r['kernels'].items()})"
  done
done
