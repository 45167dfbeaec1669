# full GPU round trip: -m gpu tests, smoke, bench N=1 (profiles/<tag>_*), reference arm, launch list
tag=${1:-r02n}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench_n1.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${tag}_ncu_bench.log 2>&1; echo "ncu rc=$?"
python tools/sweep.py --out gpurun_out/${tag}_sweep.json > gpurun_out/${tag}_sweep.txt 2>&1; echo "sweep rc=$?"
ncu --set full --clock-control none --import-source on -k "regex:k_softmax" -s 1 -c 1 -o /tmp/sm_${tag} -f python tools/prof_ops.py softmax > /tmp/sm_${tag}.log 2>&1
python tools/ncu_summary.py /tmp/sm_${tag}.ncu-rep gpurun_out/${tag}_softmax_full.txt > /dev/null 2>&1; echo "ncu full rc=$?"
