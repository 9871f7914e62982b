uname -m; nproc; lscpu | head -20; nvidia-smi; python -c "import numba, numpy; print(numba.__version__, numpy.__version__)"; python -c "import numpy as np; np.show_config()" 2>&1 | tail -30; free -g
