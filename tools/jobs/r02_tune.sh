for A in 6 8; do RMPC_SHARED_AGENTS=$A timeout 600 python tools/time_solve.py 16384 2 3 4 5 6 8 10 12 16 20 24 32; done
