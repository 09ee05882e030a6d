"""pytest plugin: `python -m pytest -p paper_2506_17626_b200.pytest_plugin <featlsq tests>`
runs featlsq's own test files unmodified against the drop-in.
`integrate.enable()` runs at configure time, before any test module does
`from featlsq.<module> import <name>`."""


def pytest_configure(config):
    from paper_2506_17626_b200 import integrate
    integrate.enable()


def pytest_report_header(config):
    import featlsq.filtering
    mod = featlsq.filtering.filter_system.__module__
    return f"featlsq stage functions -> {mod.split('.')[0]}"
