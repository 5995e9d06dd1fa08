run() { timeout 60 python tools/quick_time.py $1 2>&1 | grep "route=transform" | head -1 | sed 's/.*b2b=/b2b=/;s/resid=[0-9.e-]* //'; }
echo "C4 base (t1=512,t2=512)"; run C4
echo "C4 t1=384 t2=512"; PA_FORCE_T1=384 run C4
echo "C4 t1=384 t2=320"; PA_FORCE_T1=384 PA_FORCE_T2=320 run C4
echo "C4 t1=256 t2=256"; PA_FORCE_T1=256 PA_FORCE_T2=256 run C4
export PA_LIB=$PWD/paper_1805_02372_b200/libpa_T640.so
echo "C4 lib640 t1=384 t2=640"; PA_FORCE_T1=384 PA_FORCE_T2=640 run C4
echo "C4 lib640 t1=640 t2=640"; PA_FORCE_T1=640 PA_FORCE_T2=640 run C4
unset PA_LIB
echo "C3 base"; run C3
echo "C3 t1=384"; PA_FORCE_T1=384 run C3
echo "C3 t1=128 t2=256"; PA_FORCE_T1=128 run C3
echo "C2 base"; run C2
echo "C2 t1=160"; PA_FORCE_T1=160 run C2
echo "C2 t1=320"; PA_FORCE_T1=320 run C2
