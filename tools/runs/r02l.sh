python tools/build.py > /dev/null 2>&1
python tools/lab/spmv_ab.py chunk4k=TOPK_CHUNK_NNZ=4096 chunk8k=TOPK_CHUNK_NNZ=8192 chunk16k=TOPK_CHUNK_NNZ=16384 chunk8kgq6=TOPK_CHUNK_NNZ=8192,TOPK_SPMV_GQ=6 chunk8kgq10=TOPK_CHUNK_NNZ=8192,TOPK_SPMV_GQ=10
