for cfg in C4 C5d C3; do
for v in "PA_FORCE_T1=512" "PA_FORCE_T1=384" "PA_FORCE_T2=320" "PA_FORCE_T2=384" "PA_FORCE_T1=384 PA_FORCE_T2=320"; do
  r=$(env $v timeout 100 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
  echo "$cfg [$v] $(echo "$r" | grep -o "'n1'.*cols_per_cta': [0-9]*") $(echo "$r" | grep -o 'b2b=.*' | sed 's/resid=[0-9.e-]* //')"
done; done
