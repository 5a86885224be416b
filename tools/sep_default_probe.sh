for shape in "sep 1024 1080 1920" "sep 16 8192 8192" "sep 256 1536 2560" "sep 4096 512 512" "sep 1024 1080 1922" "seppad 1024 1080 1920"; do python tools/perf_shape.py $shape 10; done
HARRIS_DEV=1 HARRIS_SEP_CONFIG=3 python tools/perf_shape.py sepcrop 1024 1080 1922 10
python tools/perf_shape.py sepcrop 1024 1080 1922 10
