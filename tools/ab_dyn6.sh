O=gpurun_out; mkdir -p $O; L=$O/ab_dyn6.log; : > $L
q() { echo "## $*" >> $L; env "$@" timeout 300 python tools/quick_time.py $C --reps 100 --variant "$V" >> $L 2>&1; }
C=c3
V="schedule=static"; q X=1
V="schedule=dynamic"; q X=1
C=c2b
V="schedule=dynamic,p2=128"; q X=1
V="schedule=dynamic,p2=128"; q PFT_DYN_NSEG=4
C=c1
V="schedule=static"; q X=1
V="schedule=dynamic,p2=64"; q X=1
