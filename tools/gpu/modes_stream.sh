set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_governor.py -m gpu -x -q > gpurun_out/tests_gov.log 2>&1; echo "tests rc=$?"
timeout 1200 python tools/modes_bench.py --kind qr --n 16384 --b 256 --engine stream --repeat 3 > gpurun_out/modes_qr16k_stream.jsonl 2> gpurun_out/modes_qr_stream.err; echo "qr rc=$?"
timeout 1200 python tools/modes_bench.py --kind lu --n 8192 --b 256 --engine stream --repeat 5 > gpurun_out/modes_lu8k_stream.jsonl 2> gpurun_out/modes_lu_stream.err; echo "lu rc=$?"
