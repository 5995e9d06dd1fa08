run() { PA_FORCE_PLAN=$1 timeout 60 python tools/quick_time.py $2 2>&1 | grep "route=transform" | head -1 | sed 's/.*info=//;s/.device.: 0, //;s/workspace.*b2b=/b2b=/;s/resid=[0-9.e-]* //'; }
for P in "10240,6144,2" "6144,10240,1" "5120,12288,1" "7168,8960,1" "6144,10240,2" "4096,15360,1"; do run $P C4; done
for P in "4096,1344,8" "2048,2688,4" "3072,1792,4" "2048,2688,2"; do run $P C3; done
