for lib in "" build_exp/librows8.so build_exp/librows16.so; do
  echo "== lib=${lib:-default}"
  if [ -n "$lib" ]; then export STC_LIBRARY=$PWD/$lib; else unset STC_LIBRARY; fi
  python tools/one_call.py cfg4 0 abc 3
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_pack_views -c 2 --csv python tools/one_call.py cfg4 0 abc 1 2>/dev/null | grep -E "k_pack_views" | awk -F'","' '{print $(NF-2), $NF}'
done
