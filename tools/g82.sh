# final-build evidence refresh: ncu --set full per kernel (c5_10, c3, c4_7d), launch list of one bench step
bash tools/prof.sh r2c_c5 c5_10 . 60
bash tools/prof.sh r2c_c3 c3 . 60
bash tools/prof.sh r2c_c4_7d c4_7d . 60
bash tools/launches.sh r2c_launches
gzip -f gpurun_out/r2c_c5_details.txt gpurun_out/r2c_c3_details.txt gpurun_out/r2c_c4_7d_details.txt
for f in r2c_c5 r2c_c3 r2c_c4_7d; do gzip -f gpurun_out/${f}_raw.csv; done
head -5 gpurun_out/r2c_launches_summary.txt
