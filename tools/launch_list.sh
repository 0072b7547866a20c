#!/bin/bash
# launch list (ncu gpu__time_duration of every library kernel) of one warm call: tools/launch_list.sh <config> <level> <variant> <out.csv>
python tools/one_call.py "$1" "$2" "$3" 2 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file "$4" python tools/one_call.py "$1" "$2" "$3" 2 > /dev/null 2>&1
