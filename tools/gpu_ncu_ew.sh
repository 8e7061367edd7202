mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:ew_bc4 --launch-skip 254 -c 1 -o gpurun_out/ew_bc4_div -f python tools/profile_step.py 2 graph > gpurun_out/ncu_ew.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:red_rows --launch-skip 516 -c 1 -o gpurun_out/red_rows -f python tools/profile_step.py 2 graph >> gpurun_out/ncu_ew.log 2>&1
python tools/ncu_summary.py gpurun_out/ew_bc4_div.ncu-rep > gpurun_out/ew_bc4_div.txt 2>&1
python tools/ncu_summary.py gpurun_out/red_rows.ncu-rep > gpurun_out/red_rows.txt 2>&1
cat gpurun_out/ew_bc4_div.txt gpurun_out/red_rows.txt
ncu -i gpurun_out/ew_bc4_div.ncu-rep --page details --csv 2>/dev/null | grep -i "stall\|Issue Slot\|Warp Cycles\|Eligible\|Active Warps\|Occupancy\|Throughput" | head -40
