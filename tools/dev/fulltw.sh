for f in 0 1; do
  for cfg in C2 C3 C4 C5d C5c; do
  r=$(PA_FULLTW=$f timeout 100 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg full=$f $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
  done
done
