for v in "" A B C D; do
  if [ -n "$v" ]; then export PA_LIB=$PWD/paper_1805_02372_b200/libpa_$v.so; else unset PA_LIB; fi
  echo "== variant ${v:-base}"
  timeout 120 python tools/quick_time.py C2 C3 C4 2>&1 | grep "route=transform" | awk 'NR%2==1' | sed 's/.*info=.*cold/cold/'
done
