O=gpurun_out; mkdir -p $O; L=$O/ab_streams.log; : > $L
q() { echo "## $C $V streams=$S" >> $L; timeout 100 python tools/quick_time.py $C --reps 200 --streams $S --variant "$V" >> $L 2>&1; echo "rc=$?" >> $L; }
C=c2c
S=1; V=""; q
S=2; V=""; q
S=2; V="k2_at=tail,tail_ctas=40"; q
S=2; V="k2_at=tail,tail_ctas=24"; q
S=2; V="k2_at=tail,tail_ctas=16"; q
S=2; V="k2_at=tail,tail_ctas=12"; q
S=3; V="k2_at=tail,tail_ctas=16"; q
S=2; V="k2_at=grid"; q
C=c2b
S=1; V=""; q
S=2; V=""; q
cut -c1-420 $L
