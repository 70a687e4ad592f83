mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/f_test.log 2>&1; echo EXIT=$? >> gpurun_out/f_test.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo EXIT=$? >> gpurun_out/f_smoke.log
python bench.py > gpurun_out/f_bench_c3.log 2>&1
python bench.py --workload c5 > gpurun_out/f_bench_c5.log 2>&1
python bench.py --impl reference > gpurun_out/f_bench_ref.log 2>&1
python tools/configs_12.py > gpurun_out/f_c12.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "profiled/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_forward.py > gpurun_out/f_launches.csv 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sfjit -s 11 -c 1 -o gpurun_out/f_sfjit_L8 python tools/prof_sfjit.py 8 > gpurun_out/f_ncu_l8.log 2>&1
python tools/sweep_c4.py --modes sf,sf_jt --out gpurun_out/f_c4_sf.json > gpurun_out/f_c4_sf.log 2>&1
