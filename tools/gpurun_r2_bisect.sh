# repeat the host-batch streaming parity tests (zero-copy rows over PCIe) on the shipped build
for i in $(seq 1 8); do
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "host_batches or host_dataset or stream" 2>&1 | tail -1
done
