bash profiles/ab_env.sh ab16 "metr_la pems_bay" - "PGTI_SPMM_VPL=1" "PGTI_WIN_ROWS=8" "PGTI_WIN_ROWS=8 PGTI_SPMM_VPL=1" "PGTI_SPMM_MMA=1"
