# ragged-window check + ncu --set full of the two reduction-chain kernel families inside one graph replay
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 600 python -m pytest tests/test_gpu_window.py tests/test_gpu_redchain.py -x -q > gpurun_out/pytest_win.log 2>&1; tail -2 gpurun_out/pytest_win.log
for k in redchain_rows redchain_cols red_cols4s_sum; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 3 -o gpurun_out/$k -f python tools/profile_step.py 2 graph > gpurun_out/ncu_$k.log 2>&1
python tools/ncu_summary.py gpurun_out/$k.ncu-rep > gpurun_out/$k.txt 2>&1; head -30 gpurun_out/$k.txt
ncu -i gpurun_out/$k.ncu-rep --page details --csv > gpurun_out/${k}_details.csv 2>&1
done
