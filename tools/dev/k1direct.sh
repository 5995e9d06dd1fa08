for v in 0 8 16; do
  for cfg in C2 C5a C3 C5c; do
  r=$(PA_K1_DIRECT_MINC=$v timeout 100 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg minc=$v $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
  done
done
