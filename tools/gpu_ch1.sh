mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"ew_chain8<\(int\)4>" -c 1 -o gpurun_out/ch8 -f python tools/profile_step.py 2 graph > /dev/null 2>&1
ncu -i gpurun_out/ch8.ncu-rep --page source --csv --print-source sass > gpurun_out/ch8_sass.csv 2>&1
ncu -i gpurun_out/ch8.ncu-rep --page details --csv > gpurun_out/ch8_details.csv 2>&1
gzip -f gpurun_out/ch8_sass.csv; rm -f gpurun_out/*.ncu-rep
timeout 600 python tools/bench_configs.py 10 > gpurun_out/bench_configs.jsonl 2>&1; cut -c1-220 gpurun_out/bench_configs.jsonl
