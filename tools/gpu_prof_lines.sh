ncu --set full --clock-control none --import-source on -k "regex:k_softmax" -s 1 -c 1 -o /tmp/sm -f python tools/prof_ops.py softmax > /tmp/sm.log 2>&1
ncu -i /tmp/sm.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > gpurun_out/sm_sass.csv.gz
ncu -i /tmp/sm.ncu-rep --page source --csv --print-source cuda,sass 2>&1 | gzip > gpurun_out/sm_cudasass.csv.gz
ls -la gpurun_out/
