O=gpurun_out; mkdir -p $O; L=$O/ab_ring.log; : > $L
q() { echo "## $C $V $E" >> $L; env $E timeout 100 python tools/quick_time.py $C --reps $REPS --variant "$V" >> $L 2>&1; echo "rc=$?" >> $L; }
C=c2c
REPS=200
E="PFT_DBG_NOFFT=1"; V=""; q
E="PFT_DBG_NOFFT=1"; V="k2_at=tail,tail_ctas=16"; q
E="PFT_DBG_NOFFT=1"; V="k2_at=tail,tail_ctas=8"; q
E="A=1"; V=""; q
cut -c1-600 $L
