#!/bin/bash
O=gpurun_out/t22; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_shared.py tests/test_gpu_residency.py -q -x > $O/pytest_codec.log 2>&1; echo "codec tests rc=$?"; tail -3 $O/pytest_codec.log
timeout 300 python tools/profile_codec.py > $O/codec.json 2> $O/codec.err; cat $O/codec.json
timeout 300 python tools/profile_codec.py --values 3145728 > $O/codec_small.json 2>> $O/codec.err; cat $O/codec_small.json
timeout 300 python tools/profile_codec.py --values 29360128 > $O/codec_mid.json 2>> $O/codec.err; cat $O/codec_mid.json
