# staged (shared-memory, vector-load) pack/unpack kernels + one-copy header
# parse: codec parity tests, codec bench, ncu kernel times
python -m pytest tests/test_gpu_codec.py tests/test_gpu_adapter.py -q -x -m gpu 2>&1 | tail -2
python tools/codec_bench.py > gpurun_out/codec_new.json 2>&1; cat gpurun_out/codec_new.json | tr -d '\n '; echo
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/codec_bench.py > gpurun_out/rl_codec2.csv 2>/dev/null; python tools/rooflines_agg.py "codec=gpurun_out/rl_codec2.csv"
