O=gpurun_out; mkdir -p $O; L=$O/ab_ring.log; : > $L
q() { echo "## $C $V $E" >> $L; env $E timeout 100 python tools/quick_time.py $C --reps $REPS --variant "$V" >> $L 2>&1; echo "rc=$?" >> $L; }
C=c2c
E="A=1"
REPS=4; V=""; q
REPS=200; V=""; q
REPS=200; V="k2_at=tail,tail_ctas=32"; q
REPS=200; V="k2_at=tail,tail_ctas=24"; q
REPS=200; V="k2_at=grid"; q
REPS=200; V=""; q
cut -c1-600 $L
