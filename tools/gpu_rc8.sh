mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"redchain_cols<\(int\)3, \(bool\)1" -c 1 -o gpurun_out/rc3 -f python tools/profile_step.py 2 graph > gpurun_out/ncu_rc3.log 2>&1
ncu -i gpurun_out/rc3.ncu-rep --page source --csv --print-source sass > gpurun_out/rc3_sass.csv 2>&1
ncu -i gpurun_out/rc3.ncu-rep --page details --csv > gpurun_out/rc3_details.csv 2>&1
gzip -f gpurun_out/rc3_sass.csv
rm -f gpurun_out/rc3.ncu-rep
