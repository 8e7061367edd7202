# ncu --set full of the step's dominant conv instantiation (split-K TMA conv) and of a large JIT chain, inside one graph replay
mkdir -p gpurun_out; rm -f gpurun_out/*.ncu-rep
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"OutPartial" -c 2 -o gpurun_out/conv_partial_full -f python tools/profile_step.py 2 graph > gpurun_out/ncu_partial.log 2>&1
python tools/ncu_summary.py gpurun_out/conv_partial_full.ncu-rep > gpurun_out/conv_partial_full.txt 2>&1; head -34 gpurun_out/conv_partial_full.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:ew_chain_jit --launch-skip 5 -c 2 -o gpurun_out/chain_full -f python tools/profile_step.py 2 graph > gpurun_out/ncu_chain.log 2>&1
python tools/ncu_summary.py gpurun_out/chain_full.ncu-rep > gpurun_out/chain_full.txt 2>&1; head -34 gpurun_out/chain_full.txt
