# ncu --set full of the bitonic register kernels (both forms), stall breakdown as CSV
ncu --set full --clock-control none --import-source on -k regex:bitonic_sort_reg -c 2 -o gpurun_out/bit_full -f python tools/profile_driver.py bitonic > gpurun_out/ncu_bit.log 2>&1
ncu -i gpurun_out/bit_full.ncu-rep --page raw --csv > gpurun_out/bit_raw.csv
ncu -i gpurun_out/bit_full.ncu-rep --page details --csv > gpurun_out/bit_details.csv
python tools/ncu_summary.py gpurun_out/bit_full.ncu-rep > gpurun_out/ncusum_bit.json
rm -f gpurun_out/bit_full.ncu-rep
