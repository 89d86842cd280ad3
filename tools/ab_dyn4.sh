O=gpurun_out; mkdir -p $O; L=$O/ab_dyn4.log; : > $L
q() { echo "## $*" >> $L; env "$@" timeout 300 python tools/quick_time.py $C --no-check --reps 100 --variant "$V" >> $L 2>&1; }
C=c2b
V="schedule=dynamic,p2=128"
q PFT_DYN_DEV=15
q PFT_DYN_DEV=31
q PFT_DYN_DEV=47
q PFT_DYN_DEV=15 PFT_DYN_NSEG=1
q PFT_DYN_DEV=15 PFT_DYN_NSEG=4
q PFT_DYN_DEV=15 PFT_DYN_GRID=256
q PFT_DYN_DEV=15 PFT_DYN_GRID=200
V="schedule=dynamic,p2=256"
q PFT_DYN_DEV=15
V="schedule=dynamic,p2=64"
q PFT_DYN_DEV=15
