#!/bin/bash
# A/B of library builds (ab_so/libqfs_<name>.so, tools: build.build(out=..., defines=...)) on one bench config.
#   tools/ab_bench.sh <config> <steps> name1 name2 ...   ("default" = the in-tree libqfs.so)
#   EXTRA="--starts 4" tools/ab_bench.sh ...            (more bench.py arguments)
cfg=$1; steps=$2; shift 2
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib="ab_so/libqfs_$v.so"; fi
  QFS_LIB=$lib timeout 300 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-tts $EXTRA 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$v', round(d['value'],1), round(d['ms_per_step'],3), r['kernel'], r['avg_launch_us'], {k:v['ms'] for k,v in r['kernels'].items()})"
done
