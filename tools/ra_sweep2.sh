export RA_SWEEP_SETTINGS='[[32,64,32,64],[64,128,32,64],[32,64,64,64],[64,128,64,64],[48,96,32,64],[32,64,32,32],[32,128,32,64],[128,256,32,64]]'
timeout 900 python tools/ra_sweep.py fibbatch fibbatch_s1 buildsum22 fib18 transform22 > gpurun_out/ra_sweep2.log 2>&1
export RA_SWEEP_SETTINGS='[[4,8,8,64],[32,64,32,64]]'
TRS_B200_RUNAHEAD=1 timeout 600 python tools/ra_sweep.py sortbatch sortbatch_s1 > gpurun_out/ra_sweep_sort.log 2>&1
