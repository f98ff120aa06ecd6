mkdir -p gpurun_out/prof
python bench.py --mode scan --no-extras --no-cpu-baseline --steps 5 > gpurun_out/prof/scan_bench.json 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:k_plan_cluster -s 20 -c 1 -o gpurun_out/prof/plan_cluster_c5 python bench.py --workload c5 --c5-batches 32 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_select_fast -s 5 -c 1 -o gpurun_out/prof/k2f python bench.py --no-extras --no-cpu-baseline --steps 3 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_select_scan -s 3 -c 1 -o gpurun_out/prof/k2a python bench.py --mode scan --no-extras --no-cpu-baseline --steps 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --workload c5 --c5-batches 24 --no-cpu-baseline > gpurun_out/prof/launches_c5.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv python bench.py --no-extras --no-cpu-baseline --steps 20 > gpurun_out/prof/launches_c2.csv 2>&1
ls -la gpurun_out/prof
