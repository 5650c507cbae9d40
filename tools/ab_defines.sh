#!/bin/bash
# A/B compile-time variants: rebuild libqfs.so with each define set, then bench lines.
#   tools/ab_defines.sh "-DQFS_FWD2_MINB=1;-DQFS_FWD2_MINB=2" "c4 c5" [steps] [repeats]
# (';' separates define sets; the default build is restored at the end)
mkdir -p gpurun_out
steps=${3:-20}; reps=${4:-1}
IFS=';' read -ra SETS <<< "$1"
for r in $(seq $reps); do
for d in "${SETS[@]}"; do
  QFS_NVCC_DEFINES="$d" python -c "from paper_2405_12866_b200 import build; build.build(force=True)" > /dev/null || { echo "build failed: $d"; continue; }
  for c in $2; do
    python bench.py --config $c --steps $steps --no-cpu-baseline --no-tts > gpurun_out/abd.json 2> gpurun_out/abd.err
    python -c "import json; d=json.loads(open('gpurun_out/abd.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$c', '$d', round(d['value'],1), round(d['ms_per_step'],3), 'ms', {k:(v['launches'],round(v['ms'],3)) for k,v in r['kernels'].items()})" || tail -3 gpurun_out/abd.err
  done
done
done
python -c "from paper_2405_12866_b200 import build; build.build(force=True)" > /dev/null
