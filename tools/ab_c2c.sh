O=gpurun_out; mkdir -p $O; L=$O/ab_c2c.log; : > $L
q() { echo "## $C $V" >> $L; timeout 300 python tools/quick_time.py $C --reps 200 --variant "$V" $P >> $L 2>&1; }
C=c2c; P=""
for V in "k2_at=grid" "k2_at=fused" "k2_at=tail" "k2_at=tail,tail_ctas=128"; do q; done
C=c2c; P="--p 65536"
for V in "k2_at=grid" "k2_at=fused"; do q; done
C=c2c; P="--p 16384"
for V in "k2_at=grid" "k2_at=fused"; do q; done
