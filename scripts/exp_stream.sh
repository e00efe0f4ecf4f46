timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_bench_contract.py tests/test_gpu_parity.py -q -x -k "peer or bench or merger or merge" > gpurun_out/m_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/m_pytest.log
timeout 300 python scripts/stream_ring_bench.py 2147483648 524288:256 2>&1 | tail -1
PASTA_STREAM_DEFER_LAUNCH=1 timeout 300 python scripts/stream_ring_bench.py 2147483648 524288:4096 2>&1 | tail -1
PASTA_STREAM_DEFER_LAUNCH=1 timeout 300 python scripts/stream_ring_bench.py 2147483648 4194304:512 2>&1 | tail -1
