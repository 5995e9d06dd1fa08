# bench + ncu launch list + ncu full capture of the three route-(a) kernels (C2)
set -o pipefail
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --steps 3 --warmup 1 --no-sweep --no-cpu > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2.csv \
    python bench.py --steps 3 --warmup 1 --no-sweep --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k[123]_" -s 6 -c 3 -o gpurun_out/prof_C2 \
    python bench.py --steps 3 --warmup 1 --no-sweep --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
