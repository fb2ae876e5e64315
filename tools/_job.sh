{
for mc in 8 32; do
  for lanes in 8 16; do
    echo "== CUDA_DEVICE_MAX_CONNECTIONS=$mc block 32 lanes $lanes"
    CUDA_DEVICE_MAX_CONNECTIONS=$mc python tools/lane_bench.py 2 32 $lanes 12 2>&1 | tail -1
  done
done
} > gpurun_out/r2_lane_bench8.txt 2>&1
{
for pin in 1 0; do
  echo "== cfg5 LAMG_NO_L2_PIN=$pin"
  LAMG_NO_L2_PIN=$pin python bench.py --config 5 --steps 1 --warmup 1 --lanes 1 --no-cpu-baseline 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); c = d['config']
        print('single ms', c['single_rhs_solve_ms'], 'cycles', c['single_rhs_cycles'], 'block ms/step', d['ms_per_step'], 'setup', c['setup_s'])
    elif 'rror' in l: print(l.strip())
"
  echo "== cfg4 LAMG_NO_L2_PIN=$pin"
  LAMG_NO_L2_PIN=$pin python bench.py --config 4 --steps 1 --warmup 1 --lanes 1 --no-cpu-baseline 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); c = d['config']
        print('single ms', c['single_rhs_solve_ms'], 'cycles', c['single_rhs_cycles'], 'block ms/step', d['ms_per_step'], 'setup', c['setup_s'])
    elif 'rror' in l: print(l.strip())
"
done
} > gpurun_out/r2_l2pin.txt 2>&1
