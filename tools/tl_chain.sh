# PDL-chain timelines under the PFT_TIMELINE variant (tools/build_variants.sh tl:PFT_TIMELINE)
IFS=';' read -ra CASES <<< "${TL_CASES:-c2b 5 148;c4 5 148}"
for a in "${CASES[@]}"; do echo "=== $a"; PFT_LIB=variants/lib_tl.so python tools/timeline3.py $a 2>&1 | grep -v Warn; done
