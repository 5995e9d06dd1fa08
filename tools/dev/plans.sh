# plan sweep: usage bash tools/dev/plans.sh > gpurun_out/plans.log
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/quick_time.py C2 C3 C4 2>&1 | grep "route=transform" | sed 's/workspace.*create/create/' | awk 'NR%2==1'
for P in ${C4PLANS:-"9600,6250,2" "12000,5000,2" "6000,10000,1" "4800,12500,1"}; do PA_FORCE_PLAN=$P timeout 60 python tools/quick_time.py C4 2>&1 | grep "route=transform" | head -1 | sed 's/workspace.*create/create/'; done
for P in ${C3PLANS:-"4096,1344,4" "2048,2688,4" "8192,672,8" "3072,1792,8" "1536,3584,2"}; do PA_FORCE_PLAN=$P timeout 60 python tools/quick_time.py C3 2>&1 | grep "route=transform" | head -1 | sed 's/workspace.*create/create/'; done
for P in ${C2PLANS:-"2240,280,8" "1120,560,8" "640,980,8" "4480,140,16"}; do PA_FORCE_PLAN=$P timeout 60 python tools/quick_time.py C2 2>&1 | grep "route=transform" | head -1 | sed 's/workspace.*create/create/'; done
