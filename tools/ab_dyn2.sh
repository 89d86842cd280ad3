O=gpurun_out; mkdir -p $O; L=$O/ab_dyn2.log; : > $L
q() { echo "## $*" >> $L; env "$@" timeout 300 python tools/quick_time.py $C --no-check --reps 100 --variant "$V" >> $L 2>&1; }
C=c2b
V="schedule=static"; q X=1
V="schedule=dynamic"; q X=1
V="schedule=dynamic,p2=128"; q X=1
V="schedule=dynamic,p2=128"; q PFT_DYN_GRID=148 PFT_DYN_NSEG=1
C=c2c
V="schedule=static"; q X=1
V="schedule=dynamic"; q X=1
C=c4
V="schedule=static"; q X=1
V="schedule=dynamic"; q X=1
