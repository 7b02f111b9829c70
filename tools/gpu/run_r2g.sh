cp variants/lib_stats.so paper_2501_07056_b200/libmagnus_b200.so
timeout 600 python tools/ncu_case.py 20 16 2>&1 | grep "\[bd\]" | tail -4
