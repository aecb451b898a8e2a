O=gpurun_out; mkdir -p $O
for cfg in "exact 1" "exact 0" "perfo 1" "perfo 0"; do set -- $cfg
 SPEC=$1 HPAC_STREAM_PAIR=$2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:bs_stream -s 1 -c 1 -o $O/r02h_bs_$1_p$2 -f python tools/exp/bs_one.py > /dev/null 2>&1
 ncu -i $O/r02h_bs_$1_p$2.ncu-rep --page details --csv > $O/r02h_bs_$1_p$2_details.csv
 ncu -i $O/r02h_bs_$1_p$2.ncu-rep --page raw --csv > $O/r02h_bs_$1_p$2_raw.csv
 rm -f $O/r02h_bs_$1_p$2.ncu-rep
done
