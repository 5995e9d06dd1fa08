run() { PA_FORCE_PLAN=$1 timeout 60 python tools/quick_time.py $2 2>&1 | grep "route=transform" | head -1 | sed 's/.*b2b=/b2b=/;s/resid=[0-9.e-]* //'; }
echo "base C4"; run 12288,5120,2 C4
echo "T768 lib, t2=768, t1=768"; PA_LIB=$PWD/paper_1805_02372_b200/libpa_T768.so PA_FORCE_T1=768 PA_FORCE_T2=768 run 12288,5120,2 C4
echo "T768 lib, t2=384, t1=384"; PA_LIB=$PWD/paper_1805_02372_b200/libpa_T768.so PA_FORCE_T1=384 PA_FORCE_T2=384 run 12288,5120,2 C4
echo "T1024 lib r8, 1024"; PA_LIB=$PWD/paper_1805_02372_b200/libpa_T1024.so PA_FORCE_T1=1024 PA_FORCE_T2=1024 run 12288,5120,2 C4
echo "base C3 4096x1344"; run 4096,1344,4 C3
echo "T768 C3 t2=384 t1=384"; PA_LIB=$PWD/paper_1805_02372_b200/libpa_T768.so PA_FORCE_T1=384 PA_FORCE_T2=384 run 4096,1344,4 C3
echo "T1024 r8 C3 t=512"; PA_LIB=$PWD/paper_1805_02372_b200/libpa_T1024.so PA_FORCE_T1=512 PA_FORCE_T2=512 run 4096,1344,4 C3
echo "base C2"; run 2240,280,8 C2
echo "T1024 r8 C2 t=512"; PA_LIB=$PWD/paper_1805_02372_b200/libpa_T1024.so PA_FORCE_T1=512 PA_FORCE_T2=512 run 2240,280,8 C2
