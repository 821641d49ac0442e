timeout 900 python tools/debug_vgg.py 2 2>&1 | tail -50
