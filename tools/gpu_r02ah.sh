# round 2, call ah: ncu --set full with source of the shipped attention backward (32K case), after the same
# command exited 0 without ncu; export the SASS-level source page (stall reasons per instruction)
set -x
D=gpurun_out/r02ah
mkdir -p $D
timeout 300 python tools/attn_bwd_ab.py > $D/plain.jsonl 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -c 1 -o $D/attn_bwd python tools/attn_bwd_ab.py > $D/ncu.log 2>&1
ncu -i $D/attn_bwd.ncu-rep --page source --csv --print-source sass > $D/source_sass.csv 2> $D/source.err
ncu -i $D/attn_bwd.ncu-rep --page raw --csv > $D/raw.csv 2>> $D/source.err
ncu -i $D/attn_bwd.ncu-rep --page details --csv > $D/details.csv 2>> $D/source.err
ls -la $D; gzip -f $D/source_sass.csv $D/raw.csv
S=$(stat -c %s $D/attn_bwd.ncu-rep); if [ "$S" -gt 30000000 ]; then rm $D/attn_bwd.ncu-rep; fi
tail -3 $D/ncu.log
