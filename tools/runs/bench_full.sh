# the driver's round-end commands: default bench line, the reference arm, smoke
python bench.py > gpurun_out/bench_r1h.log 2> gpurun_out/bench_r1h.err
tail -c 400 gpurun_out/bench_r1h.err
python bench.py --impl reference > gpurun_out/bench_ref_r1h.log 2>&1
tail -1 gpurun_out/bench_ref_r1h.log | cut -c1-300
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
