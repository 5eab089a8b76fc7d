for cfg in 2 3 4; do timeout 120 python tools/prof_solve.py $cfg 1 2>&1 | grep -o '"max_program_block": [0-9.]*, "staged_program_capacity": [0-9.]*\|"program_bytes": [0-9.e+]*'; done
