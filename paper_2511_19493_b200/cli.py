"""The reference's ``rfx`` command line with the B200 proximity path.

    python -m paper_2511_19493_b200.cli [--device cuda] proximity --backend lowrank ...
    python -m paper_2511_19493_b200.cli mds --prox lr.rfxq ...

The commands, options and output files are the reference's own
(``rfx.cli``, cli.py:88-460: ``proximity`` :188-266, ``mds`` :269-295,
``outliers`` :298-317, ``viz-export`` :320-417); ``rfx_compat.install``
patches the proximity / MDS functions they call (``proximity_mod.*``,
``mds_mod.*`` are looked up at call time), so ``rfx proximity`` and
``rfx mds`` compute on the GPU and write byte-compatible RFXP / RFXT / RFXQ
files through the reference writers (proximity.py:602-751).  ``--device
cpu`` runs the reference unchanged.  The reference package must be importable
(``baseline/_ref`` or ``/root/reference/pkg/src``).
"""

from __future__ import annotations

import sys

from . import rfx_compat


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    device = "cuda"
    if argv[:1] == ["--device"] and len(argv) > 1:
        device, argv = argv[1], argv[2:]
    elif argv and argv[0].startswith("--device="):
        device, argv = argv[0].split("=", 1)[1], argv[1:]
    if device not in ("cuda", "cpu"):
        print(f"--device must be cuda or cpu, got {device!r}", file=sys.stderr)
        return 2
    rfx = rfx_compat.import_reference()
    import rfx.cli
    if device == "cuda":
        rfx_compat.install(rfx)
    try:
        rfx.cli.main.main(args=argv, prog_name="rfx", standalone_mode=False)
    except SystemExit as e:  # click exits with the command's status
        return int(e.code or 0)
    except Exception as e:  # noqa: BLE001 - the reference CLI's error contract
        import click
        if isinstance(e, click.ClickException):
            e.show()
            return e.exit_code
        raise
    finally:
        if device == "cuda":
            rfx_compat.uninstall(rfx)
    return 0


if __name__ == "__main__":
    sys.exit(main())
