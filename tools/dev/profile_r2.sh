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
# reduce on the box (gpurun returns at most 64 MiB): summaries, SASS stall tables and
# per-instruction shared-memory wavefronts; only the C4 report itself comes back
for c in C4 C3 C2 C1_batched; do
  python tools/ncu_summary.py gpurun_out/r2/prof_$c.ncu-rep --json gpurun_out/r2/ncu_$c.json > /dev/null 2>&1
done
rm -f gpurun_out/r2/stalls.txt
for ck in C4:k1p_fwd C4:k2_rows_t C4:k3_inv C4:k0_bits C1_batched:k_toeplitz_bitpacked; do
  c=${ck%%:*}; k=${ck#*:}
  ncu -i gpurun_out/r2/prof_$c.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/r2/src_$k.csv 2>/dev/null
  echo "== $k ($c, ncu --set full, SASS opcode aggregation: share of stall samples / of executed warp instructions, top stall reasons)" >> gpurun_out/r2/stalls.txt
  python tools/ncu_sass_stalls.py gpurun_out/r2/src_$k.csv 14 >> gpurun_out/r2/stalls.txt 2>&1
  echo >> gpurun_out/r2/stalls.txt
  rm -f gpurun_out/r2/src_$k.csv
done
python tools/dev/smem_lines.py gpurun_out/r2/prof_C4.ncu-rep "k1p|k2_rows|k3_inv|k0_bits" 6 > gpurun_out/r2/smem_lines_C4.txt 2>&1
rm -f gpurun_out/r2/prof_C3.ncu-rep gpurun_out/r2/prof_C2.ncu-rep gpurun_out/r2/prof_C1_batched.ncu-rep
du -sh gpurun_out
