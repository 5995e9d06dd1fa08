run() { timeout 60 python tools/quick_time.py $1 2>&1 | grep "route=transform" | head -1 | sed 's/.*info=//;s/.device.: 0, //;s/workspace.*b2b=/b2b=/;s/resid=[0-9.e-]* //;s/.n.: [0-9]*, .m.: [0-9]*, .route.: 1, //'; }
echo base; run C2
echo "r8 t512"; PA_MAXRADIX=8 run C2
echo "r4 t512"; PA_MAXRADIX=4 run C2
export PA_LIB=$PWD/paper_1805_02372_b200/libpa_T1024.so
echo "r4 t1024 lib1024"; PA_MAXRADIX=4 PA_FORCE_T1=1024 PA_FORCE_T2=1024 run C2
echo "r8 t1024 lib1024"; PA_MAXRADIX=8 PA_FORCE_T1=1024 PA_FORCE_T2=1024 run C2
echo "r4 t512 lib1024"; PA_MAXRADIX=4 PA_FORCE_T1=512 PA_FORCE_T2=512 run C2
echo "r4 t1024 C3"; PA_MAXRADIX=4 PA_FORCE_T1=1024 PA_FORCE_T2=1024 run C3
unset PA_LIB
echo "base C3"; run C3
