# Same-box sweep of developer overrides (one quick_time.py run per config x variant).
#   CFGS="C2 C4" bash tools/dev/env_sweep.sh "" "PA_FORCE_PLAN=4096,160,16" "PA_K3T=1 PA_LR=1"
# Developer overrides read by the library (route_a.cu ra_plan unless noted; none is needed in use):
#   PA_FORCE_PLAN=N1,N2,C   PA_FORCE_T1/T2=threads   PA_FORCE_RMAX1=8 (row-plan radix cap)
#   PA_PF=0|d (K2 row prefetch distance)   PA_PFS=0|1 (K2 own-spectrum prefetch)
#   PA_K1_DIRECT_MINC=c (K1 key gather)    PA_K1_GOUT_MINC=c (K1 direct stores)   PA_K1_BITS=0
#   PA_K13_ASC=0 (default radix order)     PA_K3_HALF=0   PA_K0_RB / PA_K0_CB (K0 tile)
#   PA_K2_T=0 / PA_K13_T=0 (general kernels)   PA_K3T=1 (TMEM-staged K3)   PA_LR=1 (row blocks)
#   PA_HOST_COPY_MAX=bytes (pa_api.cu: pa_hash_host copy kernels up to this key size; 0 = engines)
for cfg in ${CFGS:-C2 C3 C4}; do
  for v in "$@"; do
    r=$(env $v timeout 120 python tools/quick_time.py $cfg 2>&1 | grep "route=transform" | head -1)
    echo "$cfg [$v] $(echo "$r" | grep -o "'n1'.*cols_per_cta': [0-9]*") $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
  done
done
