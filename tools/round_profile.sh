#!/bin/bash
# One GPU session: tests, smoke, the default bench line, the other configs, the
# sample-sharded / emulated-exchange lines, the ncu launch list, full ncu
# captures of the dominant kernels (streamed bwd at C4, resident sweep at C3)
# and DRAM traffic per launch.  Every step under its own timeout.  Outputs
# under gpurun_out/.
set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 300 --timeout_method thread \
  > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log; grep FAILED gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 3000 gpurun_out/bench_c4.json
summ() {
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']; print(sys.argv[2], round(d['value'],1), d['unit'], round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), r['kernel'], 'frac', r['frac'], r['unit'], 'clocks', d['clocks'], 'tts', d['time_to_solution'])" "$1" "$2"
}
# short-sweep configs: 50 steps, so the per-call fixed cost (gate upload / download,
# ~0.1-0.25 ms, tools/step_overhead.py) and timer noise stay small against the timed region
for c in c2 c3 c5 c5b c5c; do
  st=50; [ $c = c5 ] && st=10
  timeout 600 python bench.py --config $c --steps $st --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  summ gpurun_out/bench_$c.json $c || tail -3 gpurun_out/bench_$c.err
done
timeout 600 python bench.py --shard sample --steps 5 --no-cpu-baseline > gpurun_out/bench_c5_sample.json 2> gpurun_out/bench_c5_sample.err
summ gpurun_out/bench_c5_sample.json c5-sample1 || tail -3 gpurun_out/bench_c5_sample.err
timeout 600 python bench.py --config c5 --emulate-ranks 8 --steps 5 --no-cpu-baseline > gpurun_out/bench_c5_emul8.json 2> gpurun_out/bench_c5_emul8.err
summ gpurun_out/bench_c5_emul8.json c5-emul8 || tail -3 gpurun_out/bench_c5_emul8.err
timeout 600 python tools/xchg_bench.py c5 10 > gpurun_out/xchg_c5.jsonl 2>/dev/null; cat gpurun_out/xchg_c5.jsonl
for s in 8; do
  timeout 600 python bench.py --config c5 --starts $s --steps 5 --no-cpu-baseline --no-tts > gpurun_out/bench_c5_s$s.json 2> gpurun_out/bench_c5_s$s.err
  summ gpurun_out/bench_c5_s$s.json c5-s$s || tail -3 gpurun_out/bench_c5_s$s.err
done
# resident-kernel pass costs in isolation (tools/res_pass_bench.cu, built beforehand into tools/res_pass_bench.bin)
[ -x tools/res_pass_bench.bin ] && timeout 120 tools/res_pass_bench.bin > gpurun_out/res_pass_bench.txt 2>&1 && cat gpurun_out/res_pass_bench.txt
if [ -n "$NO_NCU" ]; then echo done; exit 0; fi
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bwd_kernel -s 305 -c 1 -o gpurun_out/prof_bwd \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/ncu_full.log 2>&1
timeout 300 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/bench_short_c3.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:res_sweep -s 5 -c 1 -o gpurun_out/prof_res_c3 \
    python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/ncu_res.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --cache-control none \
    --clock-control none -k regex:"bwd_kernel|fwd2_kernel|fwd_gate" -s 600 -c 6 --csv --log-file gpurun_out/traffic.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tts > gpurun_out/ncu_traffic.log 2>&1
echo done
