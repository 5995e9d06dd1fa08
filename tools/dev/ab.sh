# A/B: committed library (libpa_head.so) vs working tree (libpa.so), same box, interleaved
for rep in 1 2; do
for lib in libpa_head.so libpa.so; do
  for cfg in C2 C3 C4 C5d; do
  r=$(PA_LIB=$PWD/paper_1805_02372_b200/$lib timeout 100 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$lib $cfg $(echo "$r" | grep -o 'cold median=[0-9.]*us') $(echo "$r" | grep -o 'b2b=[0-9.]*us') $(echo "$r" | grep -o 'k2_rows=[0-9.]*us')"
  done
done; done
