python -m pytest tests/test_cli.py -q -m gpu > gpurun_out/r2_tests_c.log 2>&1; tail -3 gpurun_out/r2_tests_c.log
{
for pin in 1 0; do
  for cfg in 5 4; do
    echo "== cfg$cfg LAMG_L2_PIN=$pin"
    LAMG_RELAX_TRACE=1 LAMG_L2_PIN=$pin python bench.py --config $cfg --steps 1 --warmup 1 --lanes 1 --no-cpu-baseline 2> gpurun_out/_l2.err | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); c = d['config']
        print('single ms', c['single_rhs_solve_ms'], 'cycles', c['single_rhs_cycles'], 'block ms/step', d['ms_per_step'], 'setup', c['setup_s'])
"
    grep -m2 "L2 window" gpurun_out/_l2.err
  done
done
} > gpurun_out/r2_l2pin.txt 2>&1
MODE=validate MAX_CYCLES=8 python tools/level_profile.py 2 1 > gpurun_out/r2_level_validate.txt 2>&1
LAMG_TAIL_DEBUG=1 python tools/level_profile.py 2 32 > gpurun_out/r2_level_k32_slices.txt 2>&1
python bench.py --steps 1 --warmup 1 --lanes 1 --skip-validate --no-cpu-baseline > gpurun_out/_b1.json 2>/dev/null && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -c 3000 --csv --log-file gpurun_out/r2_ncu_launches_bench_timed_region.csv python bench.py --steps 1 --warmup 1 --lanes 1 --skip-validate --no-cpu-baseline > gpurun_out/_ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/r2_ncu_launches_bench_timed_region.csv 25 > gpurun_out/r2_ncu_launches_bench_timed_region.txt 2>&1
gzip -f gpurun_out/r2_ncu_launches_bench_timed_region.csv
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:bgs_exact -c 1 -o gpurun_out/r2_ncu_full_bgs_exact python tools/batch_timing.py 2 32 2 3 > gpurun_out/_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:tail_kernel -c 1 -o gpurun_out/r2_ncu_full_tail_kernel python tools/batch_timing.py 2 32 2 3 > gpurun_out/_ncu3.log 2>&1
ls -la gpurun_out/*.ncu-rep
