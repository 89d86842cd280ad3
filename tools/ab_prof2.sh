O=gpurun_out; mkdir -p $O
export PFT_DYN_DEV=7
python tools/prof_one.py c2b "schedule=dynamic,p2=128" 3 > $O/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k1d_contract -s 1 -c 1 -o $O/prof_k1d7_c2b python tools/prof_one.py c2b "schedule=dynamic,p2=128" 3 > $O/prof_ncu.log 2>&1
unset PFT_DYN_DEV
timeout 900 ncu --set full --clock-control none -k regex:k1_contract -s 1 -c 1 -o $O/prof_k1s2_c2b python tools/prof_one.py c2b "schedule=static" 3 >> $O/prof_ncu.log 2>&1
ls -la $O | tail -4
