for v in "" "PA_FORCE_PLAN=4096,160,8 PA_FORCE_T1=128" "PA_FORCE_PLAN=4096,160,8 PA_FORCE_T1=160" "PA_FORCE_PLAN=4096,160,4 PA_FORCE_T1=64" "PA_FORCE_PLAN=4096,160,16 PA_FORCE_T1=160" "PA_FORCE_PLAN=4096,160,16 PA_FORCE_T1=128"; do
  r=$(env $v timeout 60 python tools/quick_time.py C2 2>&1 | grep "route=transform" | head -1)
  echo "[$v] $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
done
