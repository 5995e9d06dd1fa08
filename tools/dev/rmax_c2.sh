for cfg in C2 C5a C3; do
for v in "" "PA_FORCE_RMAX1=8 PA_FORCE_T2=512" "PA_FORCE_RMAX1=8"; do
  r=$(env $v timeout 60 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg [$v] $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
done; done
