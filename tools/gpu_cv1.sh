mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep
timeout 400 python tools/conv_table.py > gpurun_out/conv_table.txt 2>&1; tail -28 gpurun_out/conv_table.txt
# the 3x3 64->64 @56 fprop and a 1x1 256->64 @56 fprop, full sets with source
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tma_conv -c 1 -o gpurun_out/cv_33 -f python tools/conv_once.py 32 64 56 56 64 3 1 1 > /dev/null 2>&1
ncu -i gpurun_out/cv_33.ncu-rep --page source --csv --print-source sass > gpurun_out/cv_33_sass.csv 2>&1
ncu -i gpurun_out/cv_33.ncu-rep --page details --csv > gpurun_out/cv_33_details.csv 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tma_conv -c 1 -o gpurun_out/cv_11 -f python tools/conv_once.py 32 256 14 14 1024 1 1 0 > /dev/null 2>&1
ncu -i gpurun_out/cv_11.ncu-rep --page source --csv --print-source sass > gpurun_out/cv_11_sass.csv 2>&1
ncu -i gpurun_out/cv_11.ncu-rep --page details --csv > gpurun_out/cv_11_details.csv 2>&1
gzip -f gpurun_out/cv_33_sass.csv gpurun_out/cv_11_sass.csv
rm -f gpurun_out/*.ncu-rep
