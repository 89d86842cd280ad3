O=gpurun_out; mkdir -p $O; L=$O/ab_dyn.log; : > $L
q() { echo "## $*" >> $L; env "$@" timeout 300 python tools/quick_time.py c2b --no-check --reps 100 --variant "$V" >> $L 2>&1; }
V="schedule=static"; q X=1
V="schedule=static,p2=256"; q X=1
V="schedule=dynamic"; q X=1
V="schedule=dynamic"; q PFT_DYN_NSEG=1
V="schedule=dynamic"; q PFT_DYN_NSEG=4
V="schedule=dynamic"; q PFT_DYN_GRID=148
V="schedule=dynamic"; q PFT_DYN_GRID=148 PFT_DYN_NSEG=1
V="schedule=dynamic,p2=128"; q X=1
V="schedule=dynamic,p2=128"; q PFT_DYN_NSEG=1
V="schedule=dynamic,p2=128"; q PFT_DYN_GRID=148 PFT_DYN_NSEG=1
V="schedule=dynamic,p2=256"; q X=1
