O=gpurun_out; mkdir -p $O; L=$O/ab_c2c_sum.log; : > $L
q() { echo "## $C $P $V" >> $L; timeout 300 python tools/quick_time.py $C --reps 100 --variant "$V" $P >> $L 2>&1; }
C=c2c
P="--p 32768"; V="k2_at=grid"; q
P="--p 16384"; for V in "second_pass=sum" "second_pass=sum,tail_ctas=64" "second_pass=sum,tail_ctas=160" "second_pass=sum,p2=64" "second_pass=sum,p2=256"; do q; done
P="--p 32768"; for V in "second_pass=sum" "second_pass=sum,p2=128"; do q; done
