# round-end check: GPU suite, smoke, default bench line, reference arm
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_r1i.log 2> gpurun_out/bench_r1i.err
tail -c 300 gpurun_out/bench_r1i.err
python bench.py --impl reference > gpurun_out/bench_ref_r1i.log 2>&1
tail -1 gpurun_out/bench_ref_r1i.log | cut -c1-200
