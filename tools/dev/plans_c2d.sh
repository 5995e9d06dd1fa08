for p in "" 5120,128,16 5120,128,8 5120,128,4 6400,104,8 5376,120,16; do
  for cfg in C2; do
  r=$(PA_FORCE_PLAN=$p timeout 60 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg plan=[$p] $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
  done
done
