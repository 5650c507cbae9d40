#!/bin/bash
# A/B a runtime switch: bench lines of several configs with ENV=value settings.
#   tools/ab_env.sh "QFS_PDL=0 QFS_PDL=1" "c4 c3 c2" [steps]
mkdir -p gpurun_out
steps=${3:-20}
for c in $2; do
  for e in $1; do
    env $e python bench.py --config $c --steps $steps --no-cpu-baseline --no-tts > gpurun_out/ab_${c}_${e}.json 2> gpurun_out/ab_${c}_${e}.err
    python -c "import json; d=json.loads(open('gpurun_out/ab_${c}_${e}.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$c', '$e', round(d['value'],1), round(d['ms_per_step'],3), 'ms', {k:(v['launches'],v['ms']) for k,v in r['kernels'].items()}, 'bwd_us', r['avg_launch_us'])" || tail -3 gpurun_out/ab_${c}_${e}.err
  done
done
