cd tools/micro
./gather2
ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors.sum,gpu__time_duration.sum --clock-control none --csv --log-file ../../gpurun_out/micro2.csv ./gather2 > /dev/null 2>&1
python ../metrics_csv.py ../../gpurun_out/micro2.csv
