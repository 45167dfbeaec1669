#!/bin/bash
# ncu --set full captures of the hot kernels (one launch each, after a warm-up), summarised into
# gpurun_out/<tag>_<op>_full.txt by tools/ncu_summary.py; the .ncu-rep files stay in /tmp (size).
# usage (on the GPU box): bash tools/prof_set.sh <tag>
tag=${1:-r02}
run() {  # $1 op name for prof_ops.py, $2 kernel regex, $3 out name
    ncu --set full --clock-control none --import-source on -k "regex:$2" -s 1 -c 1 -o /tmp/$3 -f \
        python tools/prof_ops.py $1 > /tmp/$3.log 2>&1
    python tools/ncu_summary.py /tmp/$3.ncu-rep gpurun_out/${tag}_$3_full.txt > /dev/null 2>&1
    echo "$3: $(grep -m1 duration_s gpurun_out/${tag}_$3_full.txt)"
}
run softmax k_softmax softmax
run gelu k_groups gelu
run ln k_ln_fused ln
run relu k_groups relu
run maxpool k_max_small maxpool
