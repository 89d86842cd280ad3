O=gpurun_out; mkdir -p $O
python tools/prof_one.py c2b "schedule=dynamic" 3 > $O/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k1d_contract -s 1 -c 1 -o $O/prof_k1d_c2b python tools/prof_one.py c2b "schedule=dynamic" 3 > $O/prof_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k1_contract -s 1 -c 1 -o $O/prof_k1s_c2b python tools/prof_one.py c2b "schedule=static" 3 >> $O/prof_ncu.log 2>&1
ls -la $O
