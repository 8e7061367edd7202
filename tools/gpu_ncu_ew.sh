mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:ew_bc4<.int.3, .int.0, .int.0>" --launch-skip 254 -c 1 -o gpurun_out/ew_bc4_div -f python tools/profile_step.py 2 graph > gpurun_out/ncu_ew.log 2>&1
python tools/ncu_summary.py gpurun_out/ew_bc4_div.ncu-rep > gpurun_out/ew_bc4_div.txt 2>&1
cat gpurun_out/ew_bc4_div.txt
ncu -i gpurun_out/ew_bc4_div.ncu-rep --page details --csv 2>/dev/null | grep -i "stall\|Issue Slot\|Warp Cycles\|Eligible\|Occupancy\|Registers\|Achieved\|L1/TEX Hit\|L2 Hit\|Mem Busy\|Max Bandwidth" | cut -d, -f12-16 | head -40
