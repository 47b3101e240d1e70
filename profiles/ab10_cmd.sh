bash profiles/ab_env.sh ab10 "pems pems_all_la" - "PGTI_SPMM_PLO=0"
