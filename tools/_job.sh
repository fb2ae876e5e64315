python -m pytest tests -m gpu -q > gpurun_out/r2_gputest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest_final.log; tail -3 gpurun_out/r2_gputest_final.log
python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench_cfg2.json 2> gpurun_out/r2_bench_cfg2.err; echo "cfg2 rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference_cfg2.json 2> gpurun_out/r2_bench_reference_cfg2.err; echo "ref2 rc=$?"
python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/r2_bench_cfg3.json 2> gpurun_out/r2_bench_cfg3.err; echo "cfg3 rc=$?"
python bench.py --config 1 --steps 3 --warmup 3 > gpurun_out/r2_bench_cfg1.json 2> gpurun_out/r2_bench_cfg1.err; echo "cfg1 rc=$?"
python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/r2_bench_cfg4.json 2> gpurun_out/r2_bench_cfg4.err; echo "cfg4 rc=$?"
python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/r2_bench_cfg5.json 2> gpurun_out/r2_bench_cfg5.err; echo "cfg5 rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -1 gpurun_out/r2_smoke.log
