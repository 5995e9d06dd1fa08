for c in 1 2 4 8; do
  for cfg in C4 C5d C3; do
  r=$(PA_CLUSTER13=$c timeout 100 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg cluster=$c $(echo "$r" | grep -o 'b2b=.*' | sed 's/resid=[0-9.e-]* //')"
  done
done
