for pf in 0 1 2 3; do
  for cfg in C4 C5d; do
  r=$(PA_PF=$pf timeout 100 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg pf=$pf $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
  done
done
