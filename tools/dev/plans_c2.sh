# C2 plan sweep: wave quantisation of K2 (rows vs 148 SMs)
for p in "" 4096,160,16 4608,144,16 4608,140,16 4320,147,16 4096,160,8 4608,144,8 2048,315,16 2048,320,16 5120,125,16 5040,125,16 3584,180,16 4704,135,16; do
  r=$(PA_FORCE_PLAN=$p timeout 60 python tools/quick_time.py C2 2>&1 | grep "route=transform" | head -1)
  echo "plan=[$p] $(echo "$r" | grep -o "'n1': [0-9]*, 'n2': [0-9]*, 'cols_per_cta': [0-9]*") $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
done
