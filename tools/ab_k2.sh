O=gpurun_out; mkdir -p $O; L=$O/ab_k2.log; : > $L
q() { echo "## $V" >> $L; timeout 300 python tools/quick_time.py $C --reps 200 --variant "$V" >> $L 2>&1; }
C=c2c
for V in "k2_at=grid" "k2_at=grid,k2_grid_ctas=128" "k2_at=grid,k2_grid_ctas=64" "k2_at=grid,k2_grid_ctas=40" "k2_at=grid,k2_grid_ctas=20" "k2_at=grid,k2_grid_ctas=10"; do q; done
C=c5
for V in "k2_at=tail" "k2_at=grid" "k2_at=grid,k2_grid_ctas=40"; do q; done
