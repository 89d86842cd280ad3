O=gpurun_out
for rep in 1 2; do
for lib in main nosplit prev; do
  if [ $lib = main ]; then unset PFT_LIB; else export PFT_LIB=variants/lib_$lib.so; fi
  for c in "c1 --p 2048" "c2b --p 16384" "c4 --p 11520"; do
    v=$(timeout 200 python bench.py --config $c --steps 1000 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2))")
    echo "$rep $lib ${c%% *} $v" >> $O/ab_libs.txt
  done
done
done
unset PFT_LIB
PFT_LIB=variants/lib_tl.so timeout 200 python tools/timeline_c3b.py > $O/tl_c3b.txt 2>&1
PFT_LIB=variants/lib_tl.so timeout 200 python tools/timeline_c3b.py 4096 64 64 4096 > $O/tl_rows2d.txt 2>&1
