for n in 7 7 6 5 5 4; do echo nraw=$n; STC_NRAW=$n timeout 100 python tools/diag_small.py "abij abef efij & a:24;b:24;i:24;j:24;e:24;f:24;" 2>&1 | grep -c "bad 0 \[\]"; done
