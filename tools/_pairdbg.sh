for d in 0; do echo "== dbg $d"; TVS_PAIR_DBG=$d timeout 120 python tools/pair_check.py 8 256 2>&1 | grep -E "watchdog|bitwise|Error:|MP/s|launches" | head -5; done
