./tools/micro/cvt_rate
python tools/skinny_malloc.py
python tools/skinny_tiles.py
python tools/trace.py ds
python tools/trace.py dsdown
