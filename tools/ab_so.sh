#!/bin/bash
# A/B prebuilt libqfs.so variants on one box: tools/ab_so.sh "a.so b.so" "c4 c5" [steps] [reps]
steps=${3:-20}; reps=${4:-1}
cp paper_2405_12866_b200/libqfs.so /tmp/libqfs_keep.so
for r in $(seq $reps); do for so in $1; do
  cp $so paper_2405_12866_b200/libqfs.so
  for c in $2; do
    python bench.py --config $c --steps $steps --no-cpu-baseline --no-tts 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', '$c', round(d['value'],1), {k:round(v['ms'],3) for k,v in d['roofline']['kernels'].items()})"
  done
done; done
cp /tmp/libqfs_keep.so paper_2405_12866_b200/libqfs.so
