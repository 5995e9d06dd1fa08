for v in 0 1; do
  for cfg in C4 C5d; do
  r=$(PA_K3T=$v timeout 100 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg k3t=$v $(echo "$r" | grep -o 'cold median=.*' )"
  done
done
