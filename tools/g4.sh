bash tools/prof.sh g4 c5_10 "sp_border_brick|sp_core_brick|lat_sort|lat_stage|lat_hist" 6 0 "sp_border_brick|sp_core_brick|lat_sort"
