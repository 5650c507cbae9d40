#!/bin/bash
# One GPU session: tests, the default bench line, other configs, ncu launch list,
# full ncu captures of the dominant kernels (streamed bwd at C4, resident sweep at
# C3) and DRAM traffic per launch.  Outputs under gpurun_out/.
set -o pipefail
mkdir -p gpurun_out
python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
python __graft_entry__.py smoke 2>&1 | tail -2
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 3000 gpurun_out/bench_c4.json
for c in c2 c3 c5 c5b c5c; do
  python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$c', round(d['value'],1), d['unit'], round(d['ms_per_step'],3), r['kernel'], 'frac', r['frac'], r['unit'], 'tts', d['time_to_solution'])" || tail -3 gpurun_out/bench_$c.err
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bwd_kernel -s 305 -c 1 -o gpurun_out/prof_bwd \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:res_sweep -s 5 -c 1 -o gpurun_out/prof_res_c3 \
    python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/ncu_res.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --cache-control none \
    --clock-control none -k regex:"bwd_kernel|fwd2_kernel|fwd_gate" -s 600 -c 6 --csv --log-file gpurun_out/traffic.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/ncu_traffic.log 2>&1
echo done
