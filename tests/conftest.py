import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (cuda:0) and the built libqcpgrad.so")


def pytest_sessionstart(session):
    # keep the in-tree library in sync with csrc/ (incremental; seconds when stale)
    from paper_2508_17522_b200.build import build

    build()
