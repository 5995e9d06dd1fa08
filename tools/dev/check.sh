timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 200 python tools/quick_time.py C2 C3 C4 2>&1 | grep "route=transform" | awk 'NR%2==1' | sed 's/workspace.*create/create/;s/cold median=[0-9.]*us ([0-9.]* Gbit\/s) //; s/resid=[0-9.e-]* //; s/m=.*device.: 0, //'
PA_FORCE_PLAN=12288,5120,2 timeout 60 python tools/quick_time.py C4 2>&1 | grep "route=transform" | head -1 | sed 's/.*b2b=/12288x5120 b2b=/'
