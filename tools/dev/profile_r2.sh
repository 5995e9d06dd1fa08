#!/bin/bash
# Round-2 evidence behind profiles/: the bench line, the ncu launch list of the bench, --set full
# captures of C4 / C3 / C2 hashes and of batched route (b), SASS stall breakdowns.
set -x
mkdir -p gpurun_out/r2
python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench rc=$?"
python bench.py --steps 3 --warmup 1 --no-sweep --no-cpu > gpurun_out/r2/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launches_C4.csv \
    python bench.py --steps 3 --warmup 1 --no-sweep --no-cpu > gpurun_out/r2/ncu_launch.log 2>&1; echo "launch rc=$?"
for c in C4 C3 C2; do
  python tools/prof_one.py $c 2 > gpurun_out/r2/plain_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k[0123]p?_" -s 4 -c 4 -o gpurun_out/r2/prof_$c \
      python tools/prof_one.py $c 2 > gpurun_out/r2/ncu_$c.log 2>&1; echo "$c rc=$?"
done
python tools/prof_batch.py C1 65535 2 > gpurun_out/r2/plain_C1b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_toeplitz_bitpacked" -s 1 -c 1 -f -o gpurun_out/r2/prof_C1_batched \
    python tools/prof_batch.py C1 65535 2 > gpurun_out/r2/ncu_C1b.log 2>&1; echo "C1b rc=$?"
./tools/dev/tmp/dmma_bench > gpurun_out/r2/dmma.txt 2>&1; echo "dmma rc=$?"
