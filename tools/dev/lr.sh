for v in 0 1; do for cfg in C4 C5d C5c C3; do
  r=$(PA_LR=$v timeout 100 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg lr=$v $(echo "$r" | grep -o 'cold median=[0-9.]*us') $(echo "$r" | grep -o 'k[123][a-z_]*=[0-9.]*us' | tr '\n' ' ')"
done; done
