mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:redchain -c 12 -o gpurun_out/rc_step -f python tools/profile_step.py 2 graph > gpurun_out/ncu_rc_step.log 2>&1
tail -2 gpurun_out/ncu_rc_step.log
python tools/ncu_summary.py gpurun_out/rc_step.ncu-rep > gpurun_out/rc_step.txt 2>&1; grep -E "^## |duration|dram read|issue active|warps active|registers|grid|block" gpurun_out/rc_step.txt | paste - - - - - - - - | cut -c1-400
