# C2 thread-count sweep (developer overrides PA_FORCE_T1 / PA_FORCE_T2)
for t2 in "" 512; do for t1 in "" 128 512; do
  r=$(PA_FORCE_T1=$t1 PA_FORCE_T2=$t2 timeout 60 python tools/quick_time.py C2 2>&1 | grep "route=transform" | head -1)
  echo "t1=[$t1] t2=[$t2] $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
done; done
