for v in 0 1; do for cfg in C4 C5d; do
  r=$(PA_K3T=$v timeout 100 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg k3t=$v $(echo "$r" | grep -o 'cold median=[0-9.]*us') $(echo "$r" | grep -o 'k3[a-z_]*=[0-9.]*us')"
done; done
