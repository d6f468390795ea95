mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; tail -c 3000 gpurun_out/bench.json
timeout 300 python tools/bench_batched.py 5 > gpurun_out/c4.log 2>&1; cat gpurun_out/c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-decode > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rsr_mv_kernel -c 1 -o gpurun_out/c2_full python tools/profile_matvec.py c2 6 float 4 > gpurun_out/ncu_c2.log 2>&1; echo ncu2 rc=$?
