O=gpurun_out; mkdir -p $O
for p in 256 512 1024 2048 4096; do
  PFT_LIB=tools/_variants/lib_tl.so timeout 120 python tools/timeline_c3.py $p 4096 >> $O/tl_c3.log 2>&1
done
for p in 256 512 1024 2048; do
  echo "p=$p" >> $O/c3_p.log
  timeout 200 python bench.py --config c3 --p $p --steps 50 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-200 >> $O/c3_p.log
done
CMD="python bench.py --config c3 --p 256 --steps 5 --warmup 3 --no-e2e --no-cpu"
$CMD > $O/plain_c3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_contract -s 3 -c 1 -o $O/prof_k1_c3 $CMD > $O/ncu_c3.log 2>&1
ls $O
