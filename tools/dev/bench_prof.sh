# bench + ncu launch list + ncu full capture of the route-(a) kernels (C2)
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --steps 3 --warmup 1 --no-sweep --no-cpu > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2.csv \
    python bench.py --steps 3 --warmup 1 --no-sweep --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k[0123]_" -s 8 -c 4 -o gpurun_out/prof_C2 \
    python bench.py --steps 3 --warmup 1 --no-sweep --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
python tools/prof_one.py C4 1 > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k[0123]_" -s 4 -c 4 -o gpurun_out/prof_C4 python tools/prof_one.py C4 1 > gpurun_out/ncu_c4.log 2>&1; echo "c4 rc=$?"
python tools/prof_one.py C3 1 > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k[0123]_" -s 4 -c 4 -o gpurun_out/prof_C3 python tools/prof_one.py C3 1 > gpurun_out/ncu_c3.log 2>&1; echo "c3 rc=$?"
