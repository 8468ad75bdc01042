# Session-3 final check of the committed build: smoke, the whole GPU suite, the default bench line,
# a C5-subset line and an ncu capture of the large-N kernel on it
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/final4
mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 400 python bench.py > $O/bench_c2.jsonl 2> $O/bench_c2.err
timeout 900 python bench.py --config c5 --graphs 1000 --steps 2 --warmup 1 --no-e2e --cpu-seconds 15 > $O/bench_c5_1k.jsonl 2> $O/bench_c5_1k.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:isorank_big_kernel -s 2 -c 1 -f -o $O/prof_big \
  python bench.py --config c5 --graphs 1000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > $O/ncu_big.log 2>&1
echo done > $O/done
