timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python tools/quick_time.py C2 C3 C4 2>&1 | grep "route=transform" | sed 's/workspace.*create/create/' | awk 'NR%2==1'
