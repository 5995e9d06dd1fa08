for p in "" 1024,640,4 1024,640,8 1024,640,16 2048,320,8 1280,512,8 1280,512,4 1536,420,4 640,1024,4 512,1280,4; do
  r=$(PA_FORCE_PLAN=$p timeout 60 python tools/quick_time.py C2 2>&1 | grep "route=transform" | head -1)
  echo "plan=[$p] $(echo "$r" | grep -o 'cold median=.*' | sed 's/resid=[0-9.e-]* //')"
done
