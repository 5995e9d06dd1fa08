for v in "PA_FORCE_PLAN=1024,640,4 PA_FORCE_T2=64" "PA_FORCE_PLAN=1024,640,4 PA_FORCE_T2=128" "PA_FORCE_PLAN=2048,320,8 PA_FORCE_T2=128" "PA_FORCE_PLAN=2048,320,16 PA_FORCE_T2=128" "PA_FORCE_PLAN=1280,512,8 PA_FORCE_T2=96" "PA_FORCE_PLAN=1024,640,8 PA_FORCE_T2=64"; do
  for cfg in C2 C5a; do
  r=$(env $v timeout 60 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg [$v] $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
  done
done
