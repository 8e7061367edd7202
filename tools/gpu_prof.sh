# conv per-shape table + ncu --set full captures of the top kernels
set -x
timeout 600 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; cat gpurun_out/conv_table.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 3 -o gpurun_out/prof_conv3x3 python tools/conv_once.py > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 3 -o gpurun_out/prof_conv1x1 python tools/conv_once.py 32 256 56 56 64 1 1 0 > gpurun_out/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:red_thread -s 300 -c 3 -o gpurun_out/prof_red python tools/profile_step.py 1 > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
