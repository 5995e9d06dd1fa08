timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 200 python tools/quick_time.py ${CFGS:-C2 C3 C4} 2>&1 | grep "route=transform" | awk 'NR%2==1' | sed 's/workspace.*create/create/;s/cold median=[0-9.]*us ([0-9.]* Gbit\/s) //; s/resid=[0-9.e-]* //; s/m=.*device.: 0, //'
timeout 300 python tools/batch_time.py C5a C5b C5c C5d 2>&1 | tail -8
