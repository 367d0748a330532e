# ncu --set full of the finalisation in isolation (tools/ubench/fin_iso.cu), source view + details
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -I paper_2605_27390_b200/csrc -o /tmp/fin_iso tools/ubench/fin_iso.cu
ncu --set full --import-source on --clock-control none -k regex:fin64 -c 1 --launch-skip 2 -o gpurun_out/fin_iso /tmp/fin_iso > gpurun_out/fin_ncu.log 2>&1
ncu -i gpurun_out/fin_iso.ncu-rep --page source --csv --print-source sass > gpurun_out/fin_src.csv 2>&1
ncu -i gpurun_out/fin_iso.ncu-rep --page details --csv > gpurun_out/fin_details.csv 2>&1
