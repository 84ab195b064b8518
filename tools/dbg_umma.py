import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from test_gpu_umma import run
for layout in range(8):
    try:
        print('layout', layout, run(layout, 64, 128, 64, 32), run(layout, 64, 256, 64, 96))
    except Exception as e:
        print(layout, 'ERR', e)
