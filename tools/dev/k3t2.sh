for v in 0 1 2; do
  r=$(PA_K3T=$v timeout 100 python tools/quick_time.py C4 2>&1 | grep "route=transform" | head -1)
  echo "C4 k3t=$v $(echo "$r" | grep -o 'k3[a-z_]*=[0-9.]*us')"
done
