HS_CQ_TRACE_FINE=1 HS_CQ_TRACE_SPLIT=1 HS_CQ_TRACE=23 timeout 600 python tools/one_factor_pcg.py C4/2 > gpurun_out/s14_a.log 2>&1; grep "cq " gpurun_out/s14_a.log | head -30
