MACKO_LIB=paper_2511_13061_b200/libmacko_cuda_trace.so timeout 300 python tools/trace_corr.py 36864x12288 > gpurun_out/r12_corr.log 2>&1
MACKO_LIB=paper_2511_13061_b200/libmacko_cuda_trace.so timeout 300 python tools/trace_corr.py 11008x4096 >> gpurun_out/r12_corr.log 2>&1
grep -v Warn gpurun_out/r12_corr.log
