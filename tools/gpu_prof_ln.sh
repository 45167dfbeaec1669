ncu --set full --clock-control none --import-source on -k "regex:k_ln_blk" -s 1 -c 1 -o /tmp/lnb -f python tools/prof_ops.py ln > /tmp/lnb.log 2>&1
python tools/ncu_summary.py /tmp/lnb.ncu-rep gpurun_out/r02o_ln_blk_full.txt > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_softmax" -s 1 -c 1 -o /tmp/sm -f python tools/prof_ops.py softmax > /tmp/sm.log 2>&1
python tools/ncu_summary.py /tmp/sm.ncu-rep gpurun_out/r02o_softmax_full.txt > /dev/null 2>&1
