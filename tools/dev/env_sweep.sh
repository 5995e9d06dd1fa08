# Same-box sweep of developer overrides (one quick_time.py run per config x variant).
#   CFGS="C2 C4" bash tools/dev/env_sweep.sh "" "PA_FORCE_PLAN=4096,160,16" "PA_K3T=1 PA_LR=1"
# Overrides (route_a.cu): PA_FORCE_PLAN=N1,N2,C  PA_FORCE_T1/T2=threads  PA_FORCE_RMAX1=8
#   PA_PF=0 (K2 row prefetch off)  PA_K1_DIRECT_MINC=c  PA_K3T=1  PA_LR=1
for cfg in ${CFGS:-C2 C3 C4}; do
  for v in "$@"; do
    r=$(env $v timeout 120 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
    echo "$cfg [$v] $(echo "$r" | grep -o "'n1'.*cols_per_cta': [0-9]*") $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
  done
done
