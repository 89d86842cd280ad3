O=gpurun_out; mkdir -p $O; L=$O/ab_ring.log; : > $L
q() { echo "## $C $V $E" >> $L; env $E timeout 100 python tools/quick_time.py $C --reps $REPS --variant "$V" >> $L 2>&1; echo "rc=$?" >> $L; }
C=c2c
REPS=200
E="A=1"; V=""; q
E="A=1"; V="k2_at=grid"; q
cut -c1-600 $L
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
