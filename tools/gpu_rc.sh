mkdir -p gpurun_out
timeout 300 python tools/redchain_bench.py > gpurun_out/redchain_bench.txt 2>&1; cat gpurun_out/redchain_bench.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:redchain -s 3 -c 3 -o gpurun_out/rc_full -f python tools/redchain_bench.py > gpurun_out/ncu_rc.log 2>&1
python tools/ncu_summary.py gpurun_out/rc_full.ncu-rep > gpurun_out/rc_full.txt 2>&1; cat gpurun_out/rc_full.txt
