timeout 400 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -26 gpurun_out/conv_table.txt | cut -c1-100
PB_TMA_NOLOAD=1 timeout 400 python tools/conv_table.py > gpurun_out/conv_table_noload.txt 2>&1; tail -26 gpurun_out/conv_table_noload.txt | cut -c1-100
