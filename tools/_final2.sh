python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err; tail -c 300 gpurun_out/r02_bench_final.err
python tools/superop_roofline.py --configs c2,c3,c4,c5 --formats sell > gpurun_out/r02_superop_spmv.jsonl 2>&1
ncu --set full --clock-control none -k regex:sell_ -s 14 -c 7 -o gpurun_out/r02_c4_sell_panels python tools/superop_roofline.py --configs c4 --formats sell --iters 2 > gpurun_out/ncu2.log 2>&1
python tools/ncu_summary.py gpurun_out/r02_c4_sell_panels.ncu-rep > gpurun_out/r02_c4_sell_panels_full.txt 2>&1
rm -f gpurun_out/r02_c4_sell_panels.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:sell_series_term -s 20 -c 1 -o gpurun_out/r02_c2_sell_term python tools/profile_series.py --config c2 --format sell > gpurun_out/ncu1.log 2>&1
python tools/ncu_summary.py gpurun_out/r02_c2_sell_term.ncu-rep > gpurun_out/r02_c2_sell_term_full.txt 2>&1
